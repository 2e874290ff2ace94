// librp C ABI and the group-execution engine (see include/rp.h for the contract).
//
// Engine model (alg1 step 4; concurrency P:639-641; group-local
// completion P:485-487):
//  - every local worker owns a CUDA stream; its gradient is produced there;
//  - rp_preduce records an "arrived" event on the arriving worker's stream;
//  - the last local arriver makes its own stream wait on the other members'
//    arrival events and enqueues the fused kernel there, then every other
//    member's stream waits on the group's completion event. No host blocking,
//    no global barrier: disjoint groups run concurrently on different streams;
//  - rp_barrier_free_wait either blocks the host on the member's completion
//    event or (RP_WAIT_DEVICE) relies on stream order; when the last member
//    has waited the GG releases the group (Group Buffer pop, lock bits clear,
//    P:741-742) and the trace logs "done".
#include <cuda_runtime.h>
#include <fcntl.h>
#include <pthread.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <algorithm>
#include <new>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "rp_internal.h"

namespace rp {
namespace {
thread_local std::string t_last_error;
}

int fail(int code, const std::string& msg) {
  t_last_error = msg;
  return code;
}

}  // namespace rp

using rp::fail;

namespace {

struct WorkerSlot {
  bool local = false;
  bool bound = false;
  float* x = nullptr;
  const float* g = nullptr;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_arrive = nullptr;  // worker's inputs are ready (recorded at rp_preduce)
  cudaEvent_t ev_group = nullptr;   // completion of a group this worker launched
  cudaEvent_t ev_done = nullptr;    // this worker's group is done, in its stream order
  bool staged = false;
  rp::MemberUpdate upd{};  // the staged alg1 step 2
  bool in_group = false;  // arrived at a group and not yet waited
  int64_t seq = 0;
  int64_t delay_ns = 0;   // rp_set_compute_delay: synthetic compute per rp_lockstep_run step
};

struct ActiveGroup {
  rp_group g{};
  uint64_t members_mask = 0;
  uint64_t local_mask = 0;
  uint64_t arrived = 0;
  uint64_t waited = 0;
  bool launched = false;
  bool released = false;  // GG release done (first observed completion)
  rp::MemberUpdate u[RP_MAX_GROUP] = {};  // alg1 step 2 of each member (staged by rp_step*)
};

std::string members_str(const rp_group& g, uint64_t mask_filter = ~0ull) {
  std::ostringstream os;
  os << "[";
  bool first = true;
  for (int i = 0; i < g.size; ++i) {
    if (!((mask_filter >> g.members[i]) & 1)) continue;
    if (!first) os << ",";
    os << g.members[i];
    first = false;
  }
  os << "]";
  return os.str();
}

// Algorithmic HBM bytes per element of one member: x read + x write, g read if stepped,
// v read + write with momentum.
// intra-GPU kernel variant for bf16 replicas (RP_PREDUCE_BF16, see preduce_tma.cu)
int bf16_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RP_PREDUCE_BF16");
    v = e && *e ? std::atoi(e) : 7;  // warp-specialized, dynamic tiles (profiles/r01_split/)
  }
  return v;
}

int64_t member_bytes(const rp::MemberUpdate& u, bool bf16 = false) {
  if (bf16) return u.g ? 6 : 4;
  if (!u.g) return 8;
  return u.v ? 20 : 12;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(RP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                 \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

}  // namespace

// One Group Generator shared by all ranks of an asynchronous multi-process job
// (RP_FLAG_SHARED_GG): POSIX shared memory, process-shared mutex ("generates
// groups in a serial manner").
struct SharedGG {
  uint64_t magic;          // written last by the creator
  pthread_mutex_t mu;
  int64_t trace_n;         // global decision-trace event counter
  rp::GGState gg;
};
constexpr uint64_t kSharedMagic = 0x52505f47475f3031ull;  // "RP_GG_01"

struct rp_ctx {
  rp_config cfg{};
  bool has_gpu = false;
  std::mutex mu;
  std::condition_variable cv;
  WorkerSlot w[RP_MAX_WORLD];
  std::map<int64_t, ActiveGroup> active;
  uint64_t inflight = 0;  // engine lock vector: members of launched, un-waited groups
  rp::GGState gg{};           // private GG (single process, or replicated in lockstep)
  rp::GGState* ggp = &gg;      // the GG in use (private or shared)
  SharedGG* shm = nullptr;     // RP_FLAG_SHARED_GG
  std::string shm_name;
  int64_t trace_local_n = 0;
  cudaStream_t comm = nullptr;      // asynchronous cross-GPU launches, in GG order
  cudaStream_t aux = nullptr;       // lockstep: intra-GPU groups beside the step's cross-GPU launch
  cudaStream_t xs = nullptr;        // ... and the cross-GPU launch itself, at the greatest priority
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_xjoin = nullptr;
  std::set<int64_t> xready;         // cross GG groups whose local members all arrived
  std::set<int64_t> xlaunched;      // cross GG groups this GPU has launched
  rp_stats stats{};
  FILE* trace = nullptr;
  bool batching = false;
  std::vector<int64_t> ready;  // groups queued inside a batch
  struct Timed {
    cudaEvent_t start, stop;
    int64_t bytes_hbm, bytes_nvlink;
    bool cross;
    int64_t batch;
  };
  int64_t batches = 0;                // rp_batch_end calls (lockstep step index)
  std::vector<Timed> timed;           // recorded, not yet read
  std::vector<cudaEvent_t> event_pool;  // timing events for reuse
  // multi-GPU
  unsigned long long* flags = nullptr;     // this GPU's flag array (IPC-exported)
  float* stage = nullptr;                  // staging: one region per local worker (IPC-exported)
  int64_t stage_region = 0;                // bytes per region
  bool peers_ready = false;
  float* peer_x[RP_MAX_WORLD] = {};                 // replicas of remote workers, mapped
  unsigned long long* peer_flags[RP_MAX_GPUS] = {};  // flag arrays of the other GPUs, mapped
  float* peer_stage[RP_MAX_GPUS] = {};              // staging buffers of the other GPUs, mapped
  // optional cross-kernel item timeline (env RP_XGPU_PROFILE=path): last launch only
  rp::XItemRecord* prof = nullptr;
  unsigned long long* cta_stat = nullptr;  // RP_XGPU_PROFILE: per-CTA wait breakdown of the last launch
  int64_t prof_cap = 0, prof_items = 0;
  std::string prof_path;
  std::vector<void*> ipc_mapped;                    // cudaIpcOpenMemHandle results
  int32_t peer_pid[RP_MAX_GPUS] = {};               // process ids (NVLS descriptor sockets)
  rp::NvlsState nvls;                               // multicast objects (rp_nvls_enable)
  // cross-GPU flag tags: launches of groups with a given slot that involved both GPUs, counted
  // on each side in launch order (lockstep: step order; asynchronous: ticket order), so a tag is
  // unique per (group launch, GPU pair) and stale flags of earlier launches never match
  uint64_t pair_tag[RP_MAX_GPUS][rp::kFlagSlots][RP_MAX_GPUS] = {};
  rp::XErr* xerr = nullptr;                         // host-mapped watchdog record
  rp::XErr* xerr_dev = nullptr;                     // its device address
  unsigned long long watchdog_ns = 0;               // flag-wait limit (0 = off)
  // RP_FLAG_EMULATE: n_gpus virtual GPUs on one device (every worker local to this process)
  bool emulate = false;
  unsigned long long* vflags = nullptr;             // n_gpus flag arrays
  float* vstage = nullptr;                          // n_gpus * wpg staging regions
  rp::XTask* d_tasks = nullptr;                     // device copy of the emulated launch's tasks
  unsigned int* claim = nullptr;                    // chunk-claim counters, kXClaimWords per (virtual) GPU
};

namespace {

// Serializes Group Generator decisions across processes (no-op for a private GG,
// which the context mutex already protects). Lock order: ctx->mu, then GGLock.
struct GGLock {
  pthread_mutex_t* m;
  explicit GGLock(rp_ctx* c) : m(c->shm ? &c->shm->mu : nullptr) {
    if (m) pthread_mutex_lock(m);
  }
  ~GGLock() {
    if (m) pthread_mutex_unlock(m);
  }
};

// Append one decision-trace event; "n" orders events of all ranks (GG order).
// Caller holds ctx->mu and the GGLock.
void trace_line(rp_ctx* c, const std::string& body) {
  const int64_t n = c->shm ? c->shm->trace_n++ : c->trace_local_n++;
  if (!c->trace) return;
  std::fprintf(c->trace, "{\"n\":%lld,%s}\n", static_cast<long long>(n), body.c_str());
  std::fflush(c->trace);
}

std::string group_json(const rp_group& g) {
  std::ostringstream os;
  os << "\"seq\":" << g.seq << ",\"members\":[";
  for (int i = 0; i < g.size; ++i) os << (i ? "," : "") << g.members[i];
  os << "]";
  return os.str();
}

bool worker_ok(const rp_ctx* c, int32_t w) { return w >= 0 && w < c->cfg.world; }

int check_group(const rp_ctx* c, const rp_group* g, uint64_t* mask) {
  if (!g || g->size < 1 || g->size > RP_MAX_GROUP) return fail(RP_EINVAL, "group size out of range");
  uint64_t m = 0;
  for (int i = 0; i < g->size; ++i) {
    const int v = g->members[i];
    if (v < 0 || v >= c->cfg.world) return fail(RP_EINVAL, "group member out of range");
    if (i > 0 && v <= g->members[i - 1]) return fail(RP_EINVAL, "group members must be strictly ascending");
    m |= 1ull << v;
  }
  *mask = m;
  return RP_OK;
}

bool same_group(const rp_group& a, const rp_group& b) {
  if (a.seq != b.seq || a.size != b.size) return false;
  for (int i = 0; i < a.size; ++i)
    if (a.members[i] != b.members[i]) return false;
  return true;
}

// GG release of a completed group + trace (caller holds mu).
int release_gg_group(rp_ctx* c, int64_t seq) {
  GGLock lk(c);
  if (c->shm && !rp::gg_find(c->ggp, seq)) return RP_OK;  // another rank observed it first
  rp_group rel{};
  const int rc = rp::gg_done(c->ggp, seq, &rel);
  if (rc != RP_OK) return rc;
  trace_line(c, "\"ev\":\"done\",\"seq\":" + std::to_string(seq));
  return RP_OK;
}

cudaEvent_t timing_event(rp_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

// Enqueue ONE fused kernel for a set of ready groups whose members are all
// local (caller holds mu). The kernel runs on the stream of the lowest local
// member after every member's arrival event; every member's stream is then
// ordered after the kernel and records its own completion event.
int launch_cross(rp_ctx* c, const std::vector<int64_t>& seqs, cudaStream_t stream, int max_ctas = 0,
                 const std::vector<int64_t>& local = {});
int launch_nvls_groups(rp_ctx* c, std::vector<int64_t> seqs, cudaStream_t stream);
int pump_cross(rp_ctx* c);

// GPU subset of a group, and whether it takes the NVLS path (rp_nvls_enable).
uint32_t gpu_mask(const rp_ctx* c, const rp_group& g) {
  uint32_t m = 0;
  for (int i = 0; i < g.size; ++i) m |= 1u << (g.members[i] / c->cfg.workers_per_gpu);
  return m;
}
bool nvls_group(const rp_ctx* c, const rp_group& g) {
  return c->nvls.min_gpus > 0 && __builtin_popcount(gpu_mask(c, g)) >= c->nvls.min_gpus;
}
int open_shared_gg(rp_ctx* c);

// Does the group span GPUs (real or, with RP_FLAG_EMULATE, virtual)?
bool is_cross(const rp_ctx* c, const ActiveGroup& a) {
  return c->emulate ? __builtin_popcount(gpu_mask(c, a.g)) > 1 : a.local_mask != a.members_mask;
}

// The host-mapped watchdog record: a cross-GPU (or NVLS) flag wait that gave up.
int check_xerr(rp_ctx* c) {
  if (!c->xerr) return RP_OK;
  if (!__atomic_load_n(&c->xerr->code, __ATOMIC_ACQUIRE)) return RP_OK;
  rp::XErr e;
  std::memcpy(&e, c->xerr, sizeof(e));
  static const char* kinds[] = {"A (partial)", "B (mean)", "READY"};
  const std::string kind = e.kind >= 0 && e.kind < 3 ? kinds[e.kind] : (e.kind >= 16 ? "NVLS" : "?");
  return fail(RP_ETIMEOUT, "cross-GPU flag wait timed out after " + std::to_string(c->watchdog_ns / 1000000000ull) +
                               " s on GPU " + std::to_string(e.gpu) + ": flag " + kind + " of chunk " +
                               std::to_string(e.chunk) + " from GPU " + std::to_string(e.src) + " (slot " +
                               std::to_string(e.slot) + ") expected tag " + std::to_string(e.tag) + ", holds " +
                               std::to_string(e.seen) + " (a peer never arrived or the collective contract broke; "
                               "the replicas of this step are undefined)");
}

int launch_groups(rp_ctx* c, const std::vector<int64_t>& all_seqs) {
  if (all_seqs.empty()) return RP_OK;
  std::vector<int64_t> seqs, cross, nv;  // intra-GPU, push cross-GPU, NVLS cross-GPU
  for (int64_t q : all_seqs) {
    const ActiveGroup& a = c->active.at(q);
    (!is_cross(c, a) ? seqs : (nvls_group(c, a.g) ? nv : cross)).push_back(q);
  }
  uint64_t all = 0;
  for (int64_t q : all_seqs) {
    ActiveGroup& a = c->active.at(q);
    c->stats.lock_assertions++;
    if ((c->inflight | all) & a.local_mask)  // a member is still inside another group
      return fail(RP_ECONFLICT, "atomicity violation: members " + members_str(a.g, c->inflight | all) +
                                    " hold an unfinished group");
    all |= a.local_mask;
  }
  int launcher = __builtin_ctzll(all);
  WorkerSlot& L = c->w[launcher];
  for (int m = 0; m < RP_MAX_WORLD; ++m)
    if (((all >> m) & 1) && m != launcher) CUDA_TRY(cudaStreamWaitEvent(L.stream, c->w[m].ev_arrive, 0));
  // With cross-GPU groups in the batch the intra-GPU groups run BESIDE them: the cross launch
  // (NVLink-bound; grid capped at RP_XGPU_SPLIT CTAs, default 296 = every resident slot) is issued
  // first on its own stream, the intra-GPU launch (HBM-bound, dynamic-tile TMA kernel, one stage
  // less) on a second stream; its CTAs take SM slots next to the cross kernel's and as they free
  // up, drawing tiles at run time. Emulated GPUs (RP_FLAG_EMULATE) run the two one after the other.
  static int split_ctas = -1;
  if (split_ctas < 0) {
    const char* v = std::getenv("RP_XGPU_SPLIT");
    split_ctas = v && *v ? std::atoi(v) : 296;
  }
  // RP_SPLIT_ORDER (experiment): 0 = concurrent streams (default), 1 = the cross launch first and
  // the intra-GPU launch after it on one stream, 2 = the intra-GPU launch first
  static int split_order = -1;
  if (split_order < 0) {
    const char* v = std::getenv("RP_SPLIT_ORDER");
    split_order = v && *v ? std::atoi(v) : 0;
  }
  // Fusion (default; RP_XGPU_FUSE=0 disables): intra-GPU groups of <= 4 members (<= 16 groups) ride
  // in the cross launch as L jobs of the warp-specialized kernel, spread over its lane iterations
  // (their HBM work fills the time NVLink flag waits leave idle; a concurrent launch could not
  // co-reside with the cross kernel's shared memory anyway). Momentum steps take the register
  // kernel, which has no L jobs: they keep the separate launch.
  static int fuse_env = -1;
  if (fuse_env < 0) {
    const char* v = std::getenv("RP_XGPU_FUSE");
    fuse_env = v && *v ? std::atoi(v) : 1;
  }
  std::vector<int64_t> fused;
  if (fuse_env && !cross.empty() && nv.empty() && !seqs.empty() && split_order == 0) {
    bool ok = seqs.size() <= static_cast<size_t>(rp::kMaxXLocalGroups);
    for (int64_t q : seqs) {
      const ActiveGroup& a = c->active.at(q);
      ok = ok && a.g.size <= rp::kMaxFusedK;
      for (int i = 0; i < a.g.size; ++i) ok = ok && !(a.u[i].v && a.u[i].g);
    }
    for (int64_t q : cross) {
      const ActiveGroup& a = c->active.at(q);
      for (int i = 0; i < a.g.size; ++i) ok = ok && !(a.u[i].v && a.u[i].g);
    }
    // ... unless the intra-GPU work dominates the step (more than twice the cross part's local
    // members, e.g. the Inter step of Inter-Intra with one Head Worker per GPU): the dedicated
    // dynamic-tile kernel moves bulk HBM traffic faster than L jobs between lane iterations
    // (cfg2ii at N = 2: 33.5k fused vs 36.0k separate; cfg4: 4.0k fused vs 3.4k separate,
    // profiles/r02/sweep_fuse_2gpu.txt)
    int intra_members = 0, cross_members = 0;
    for (int64_t q : seqs) intra_members += c->active.at(q).g.size;
    for (int64_t q : cross) cross_members += __builtin_popcountll(c->active.at(q).local_mask);
    if (c->emulate) cross_members = intra_members;  // emulation: always exercise the L jobs
    if (ok && intra_members <= 2 * cross_members) fused.swap(seqs);
  }
  const bool split = !cross.empty() && nv.empty() && !seqs.empty() && !c->emulate && c->aux && c->xs &&
                     split_order == 0;
  if (!split && split_order == 1 && !cross.empty() && nv.empty() && !c->emulate) {
    const int rc = launch_cross(c, cross, L.stream);
    if (rc != RP_OK) return rc;
    cross.clear();
  }
  cudaStream_t intra_stream = L.stream;
  static int tpc = -1;  // RP_DYN_TPC: tiles per CTA of the intra-GPU launch in split mode
  if (tpc < 0) {
    const char* v = std::getenv("RP_DYN_TPC");
    tpc = v && *v ? std::atoi(v) : 0;
  }
  if (split) {
    CUDA_TRY(cudaEventRecord(c->ev_fork, L.stream));
    CUDA_TRY(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
    CUDA_TRY(cudaStreamWaitEvent(c->xs, c->ev_fork, 0));
    intra_stream = c->aux;
    const int rc = launch_cross(c, cross, c->xs, split_ctas);
    if (rc != RP_OK) return rc;
    CUDA_TRY(cudaEventRecord(c->ev_xjoin, c->xs));
  }
  // One fused launch for all remaining intra-GPU groups (chunked at kMaxTasks
  // groups / kMaxTaskMembers members).
  size_t gi = 0;
  while (gi < seqs.size()) {
    rp::MultiTask t{};
    if (split) {
      t.reserve_sms = split_ctas;  // beside a cross launch: dynamic-tile kernel, one stage less
      t.tiles_per_cta = tpc;       // retiring CTAs: the cross launch's CTAs find free slots
    }
    int nm = 0;
    int64_t bytes = 0;
    while (gi < seqs.size() && t.ngroups < rp::kMaxTasks) {
      ActiveGroup& a = c->active.at(seqs[gi]);
      if (nm + a.g.size > rp::kMaxTaskMembers) break;
      t.group_k[t.ngroups] = a.g.size;
      t.group_first[t.ngroups] = nm;
      for (int i = 0; i < a.g.size; ++i) {
        t.x[nm] = c->w[a.g.members[i]].x;
        t.u[nm] = a.u[i];
        bytes += member_bytes(a.u[i], c->cfg.dtype == RP_DTYPE_BF16) * c->cfg.n_params;
        ++nm;
      }
      t.ngroups++;
      if (a.g.size == 1) c->stats.singleton_groups++;
      c->stats.groups_launched++;
      ++gi;
    }
    const bool timing = (c->cfg.flags & RP_FLAG_TIMING) != 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) {
      e0 = timing_event(c);
      e1 = timing_event(c);
      if (!e0 || !e1) return fail(RP_ECUDA, "timing event creation failed");
      CUDA_TRY(cudaEventRecord(e0, intra_stream));
    }
    std::string err;
    const int rc = c->cfg.dtype == RP_DTYPE_BF16
                       ? rp::launch_preduce_tma(t, c->cfg.n_params, intra_stream, &err, bf16_variant(), true)
                       : rp::launch_preduce_multi(t, c->cfg.n_params, intra_stream, &err);
    if (rc != RP_OK) return fail(rc, err);
    if (timing) {
      CUDA_TRY(cudaEventRecord(e1, intra_stream));
      c->timed.push_back({e0, e1, bytes, 0, false, c->batches});
    }
    c->stats.kernel_launches++;
    c->stats.bytes_hbm += bytes;
  }
  // NVLS groups first, then the push kernel: every GPU issues its cross-GPU launches in
  // the same order, so no launch waits on a peer's later launch (split: already issued)
  if (split) {
    CUDA_TRY(cudaEventRecord(c->ev_join, c->aux));
    CUDA_TRY(cudaStreamWaitEvent(L.stream, c->ev_join, 0));
    CUDA_TRY(cudaStreamWaitEvent(L.stream, c->ev_xjoin, 0));
  } else if (!nv.empty()) {
    const int rc = launch_nvls_groups(c, nv, L.stream);
    if (rc != RP_OK) return rc;
  }
  if (!split && !cross.empty()) {
    const int rc = launch_cross(c, cross, L.stream, 0, fused);
    if (rc != RP_OK) return rc;
  }
  CUDA_TRY(cudaEventRecord(L.ev_group, L.stream));
  for (int m = 0; m < RP_MAX_WORLD; ++m) {
    if (!((all >> m) & 1)) continue;
    WorkerSlot& s = c->w[m];
    if (m != launcher) CUDA_TRY(cudaStreamWaitEvent(s.stream, L.ev_group, 0));
    CUDA_TRY(cudaEventRecord(s.ev_done, s.stream));
  }
  for (int64_t q : all_seqs) c->active.at(q).launched = true;
  c->inflight |= all;
  c->cv.notify_all();
  return RP_OK;
}

// Addresses of GPU d's objects as seen from this process: its flag array, the staging region of
// its local worker `region`, and worker m's replica (all local when emulating).
unsigned long long* flags_of(rp_ctx* c, int d) {
  if (c->emulate) return c->vflags + static_cast<size_t>(d) * rp::kFlagWords;
  return d == c->cfg.rank ? c->flags : c->peer_flags[d];
}
float* stage_of(rp_ctx* c, int d, int region) {
  char* base = c->emulate ? reinterpret_cast<char*>(c->vstage) + static_cast<int64_t>(d) * c->cfg.workers_per_gpu *
                                                                    c->stage_region
                          : reinterpret_cast<char*>(d == c->cfg.rank ? c->stage : c->peer_stage[d]);
  return base ? reinterpret_cast<float*>(base + region * c->stage_region) : nullptr;
}
float* replica_of(rp_ctx* c, int m) {
  return c->emulate || c->w[m].local ? c->w[m].x : c->peer_x[m];
}

// GPU `gpu`'s parts of the cross-GPU groups `seqs` (ascending seq: the same part order on every
// GPU), with the algorithmic bytes of those parts (caller holds mu).
int build_task(rp_ctx* c, const std::vector<int64_t>& seqs, const std::vector<int64_t>& local, int gpu,
               rp::XTask& T, int64_t* nvl_out, int64_t* hbm_out) {
  const int wpg = c->cfg.workers_per_gpu;
  T = rp::XTask{};
  T.my_gpu = gpu;
  T.n = c->cfg.n_params;
  T.my_flags = flags_of(c, gpu);
  T.bf16 = c->cfg.dtype == RP_DTYPE_BF16;
  T.watchdog_ns = c->watchdog_ns;
  T.err = c->xerr_dev;
  static int dyn = -1;  // RP_XGPU_DYN=0: static chunk -> lane assignment (comparison)
  if (dyn < 0) {
    const char* v = std::getenv("RP_XGPU_DYN");
    dyn = v && *v ? std::atoi(v) : 1;
  }
  T.claim = dyn && c->claim ? c->claim + static_cast<size_t>(c->emulate ? gpu : 0) * rp::kXClaimWords : nullptr;
  // claim order (xgpu_ws.cu): part by part when every group of the launch comes from a static
  // schedule (seq < 0), chunk-major for Group-Generator groups; RP_XGPU_CLAIM=part|chunk overrides
  static int order = -1;
  if (order < 0) {
    const char* v = std::getenv("RP_XGPU_CLAIM");
    order = !v || !*v ? 2 : (std::string(v) == "part" ? 1 : 0);
  }
  bool all_static = true;
  for (int64_t q : seqs) all_static = all_static && q < 0;
  T.part_major = order == 2 ? (all_static ? 1 : 0) : order;
  const int64_t esz = T.bf16 ? 2 : 4;  // bytes per replica element
  int64_t nvl = 0, hbm = 0;
  for (int64_t q : seqs) {
    ActiveGroup& a = c->active.at(q);
    if (!((gpu_mask(c, a.g) >> gpu) & 1)) continue;
    if (T.nparts >= rp::kMaxXParts) return fail(RP_EINVAL, "more than 8 cross-GPU groups on one GPU in one step");
    rp::XPart& p = T.part[T.nparts++];
    p.k_total = a.g.size;
    p.slot = a.g.members[0];
    int last_gpu = -1;
    for (int i = 0; i < a.g.size; ++i) {
      const int m = a.g.members[i];
      const int d = m / wpg;
      if (d != last_gpu) {  // first (lowest) member on GPU d: receives the means, owns the region
        if (p.kp >= rp::kMaxXGpus) return fail(RP_EINVAL, "group spans more than 8 GPUs");
        p.gpu[p.kp] = d;
        if (d == gpu) p.me = p.kp;
        p.xfirst[p.kp] = replica_of(c, m);
        p.stage[p.kp] = stage_of(c, d, m - d * wpg);
        p.pflags[p.kp] = flags_of(c, d);
        p.kp++;
        last_gpu = d;
      }
      if (d == gpu) {
        if (p.m >= rp::kMaxXLocal) return fail(RP_EINVAL, "more than 8 local members in a cross-GPU group");
        p.x[p.m] = c->w[m].x;
        p.u[p.m] = a.u[i];
        p.m++;
      }
    }
    for (int d = 0; d < p.kp; ++d)
      if (d != p.me) p.tag[d] = ++c->pair_tag[gpu][p.slot][p.gpu[d]];
    rp::xgpu_geometry(p, T.n);
    // NVLink bytes this GPU stores into peers: A, its partials of the other slices; B, its
    // slice's means to every peer (fp32 partials; bf16 replicas move esz = 2 bytes per element)
    const int64_t lo = std::min<int64_t>(p.me * p.S4, p.n4), hi = std::min<int64_t>((p.me + 1) * p.S4, p.n4);
    int64_t mine = 4 * (hi - lo);
    if (p.me == p.kp - 1) mine += p.rem;
    const int64_t others = T.n - mine;
    nvl += 4 * others + esz * (p.kp - 1) * mine;
    int64_t rd = 0;
    for (int m = 0; m < p.m; ++m) rd += member_bytes(p.u[m], T.bf16) - esz;  // reads (x, g, v) + v write
    // A+B reads of x,g; B reads of staged partials; B stores of xbar; C copies (m > 1)
    hbm += rd * T.n + 4 * (p.kp - 1) * mine + esz * p.m * mine + 2 * esz * (p.m - 1) * others;
  }
  for (int64_t q : local) {  // fused intra-GPU groups of this GPU (L jobs)
    ActiveGroup& a = c->active.at(q);
    if (a.g.members[0] / wpg != gpu) continue;
    rp::XLocalGroup& G = T.lg[T.nlocal++];
    G.k = a.g.size;
    for (int i = 0; i < a.g.size; ++i) {
      G.x[i] = c->w[a.g.members[i]].x;
      G.u[i] = a.u[i];
      hbm += member_bytes(a.u[i], T.bf16) * T.n;
    }
    c->stats.groups_launched++;
    if (a.g.size == 1) c->stats.singleton_groups++;
  }
  *nvl_out = nvl;
  *hbm_out = hbm;
  return RP_OK;
}

// This GPU's parts of every cross-GPU group of the batch, in ONE xgpu launch (caller holds mu;
// members' arrival events already joined into `stream`). Emulated GPUs: every virtual GPU's
// parts in ONE cooperative launch.
// RP_DEBUG_POISON=1 (race check; compute-sanitizer is closed on this pool): before a cross
// launch, fill the staging rows this GPU owns with 0xFF bytes (a NaN pattern). The peers may push
// into them only after this launch posts READY, so a B stage that read a partial before it
// arrived would fold a NaN into the mean and fail the bit-exact parity tests.
int poison_staging(const rp::XTask& T, cudaStream_t stream) {
  for (int pi = 0; pi < T.nparts; ++pi) {
    const rp::XPart& p = T.part[pi];
    const size_t bytes = static_cast<size_t>(p.kp) * static_cast<size_t>(p.S4 + 1) * 16;
    CUDA_TRY(cudaMemsetAsync(p.stage[p.me], 0xFF, bytes, stream));
  }
  return RP_OK;
}
bool poison_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RP_DEBUG_POISON");
    v = e && *e && std::atoi(e) != 0;
  }
  return v == 1;
}

int launch_cross(rp_ctx* c, const std::vector<int64_t>& seqs_in, cudaStream_t stream, int max_ctas,
                 const std::vector<int64_t>& local) {
  if (!c->peers_ready) return fail(RP_ESTATE, "cross-GPU group before rp_peer_import");
  std::vector<int64_t> seqs(seqs_in);
  std::sort(seqs.begin(), seqs.end());
  c->stats.groups_launched += static_cast<int64_t>(seqs.size());
  c->stats.cross_gpu_groups += static_cast<int64_t>(seqs.size());
  const bool timing = (c->cfg.flags & RP_FLAG_TIMING) != 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timing) {
    e0 = timing_event(c);
    e1 = timing_event(c);
    if (!e0 || !e1) return fail(RP_ECUDA, "timing event creation failed");
    CUDA_TRY(cudaEventRecord(e0, stream));
  }
  int64_t nvl = 0, hbm = 0;
  std::string err;
  if (c->emulate) {
    const int V = c->cfg.n_gpus;
    std::vector<rp::XTask> tasks(V);
    for (int d = 0; d < V; ++d) {
      int64_t a = 0, b = 0;
      const int rc = build_task(c, seqs, local, d, tasks[d], &a, &b);
      if (rc != RP_OK) return rc;
      nvl += a;
      hbm += b;
    }
    if (poison_enabled())
      for (int d = 0; d < V; ++d) {
        const int prc = poison_staging(tasks[d], stream);
        if (prc != RP_OK) return prc;
      }
    const int rc = rp::launch_xgpu_emulated(tasks.data(), V, c->d_tasks, stream, &err);
    if (rc != RP_OK) return fail(rc, err);
  } else {
    rp::XTask T;
    int rc = build_task(c, seqs, local, c->cfg.rank, T, &nvl, &hbm);
    if (rc != RP_OK) return rc;
    T.max_ctas = max_ctas;
    if (!c->prof_path.empty()) {
      const int64_t items = static_cast<int64_t>(T.nparts) * 3 * rp::kMaxChunks;
      if (items > c->prof_cap) {
        if (c->prof) cudaFree(c->prof);
        c->prof = nullptr;
        c->prof_cap = 0;
        if (cudaMalloc(&c->prof, items * sizeof(rp::XItemRecord)) == cudaSuccess) c->prof_cap = items;
      }
      T.prof = c->prof;
      c->prof_items = items;
      if (c->prof) {
        cudaMemsetAsync(c->prof, 0, items * sizeof(rp::XItemRecord), stream);
        if (!c->cta_stat) cudaMalloc(&c->cta_stat, sizeof(unsigned long long) * rp::kCtaStatWords);
        if (c->cta_stat) cudaMemsetAsync(c->cta_stat, 0, sizeof(unsigned long long) * rp::kCtaStatWords, stream);
        T.cta_stat = c->cta_stat;
      }
    }
    if (poison_enabled()) {
      rc = poison_staging(T, stream);
      if (rc != RP_OK) return rc;
    }
    rc = rp::launch_xgpu(T, stream, &err);
    if (rc != RP_OK) return fail(rc, err);
  }
  if (timing) {
    CUDA_TRY(cudaEventRecord(e1, stream));
    c->timed.push_back({e0, e1, hbm, nvl, true, c->batches});
  }
  c->stats.kernel_launches++;
  c->stats.bytes_hbm += hbm;
  c->stats.bytes_nvlink += nvl;
  return RP_OK;
}

// This GPU's parts of every NVLS group of the batch, in ONE nvls launch (caller holds mu).
// Slots: the k-th group launched on a GPU subset uses slot k mod slots with tag
// k / slots + 1; every GPU of the subset launches the subset's groups in the same order
// (ascending seq within a batch; batches in step order; asynchronous groups in ticket
// order), so all agree on slot and tag.
int launch_nvls_groups(rp_ctx* c, std::vector<int64_t> seqs, cudaStream_t stream) {
  if (!c->peers_ready) return fail(RP_ESTATE, "cross-GPU group before rp_peer_import");
  if (static_cast<int>(seqs.size()) > rp::kMaxNParts)
    return fail(RP_EINVAL, "more than 8 NVLS groups on one GPU in one step");
  std::sort(seqs.begin(), seqs.end());
  const int wpg = c->cfg.workers_per_gpu;
  rp::NTask T{};
  T.nparts = static_cast<int32_t>(seqs.size());
  const int64_t n = c->cfg.n_params;
  int64_t hbm = 0, nvl = 0;
  for (size_t pi = 0; pi < seqs.size(); ++pi) {
    ActiveGroup& a = c->active.at(seqs[pi]);
    rp::NvlsObj* o = rp::nvls_find(&c->nvls, gpu_mask(c, a.g));
    if (!o) return fail(RP_ESTATE, "no multicast object for the GPU subset of group " + std::to_string(a.g.seq));
    rp::NPart& p = T.part[pi];
    const int64_t use = o->launched++;
    const int64_t slot = use % o->slots;
    p.tag = static_cast<uint64_t>(use / o->slots) + 1;
    p.kp = o->kp;
    p.me = o->me;
    p.k_total = a.g.size;
    p.rem = static_cast<int32_t>(n % 4);
    p.n4 = n / 4;
    p.CH = o->CH;
    p.nch = o->nch;
    char* ucb = reinterpret_cast<char*>(o->uc_va) + slot * o->slot_bytes;
    char* mcb = reinterpret_cast<char*>(o->mc_va) + slot * o->slot_bytes;
    p.uc = reinterpret_cast<float*>(ucb);
    p.mc = reinterpret_cast<float*>(mcb);
    p.ucf = reinterpret_cast<unsigned long long*>(ucb + o->data_bytes);
    p.mcf = reinterpret_cast<unsigned long long*>(mcb + o->data_bytes);
    p.watchdog_ns = c->watchdog_ns;
    p.err = c->xerr_dev;
    p.gpu = c->cfg.rank;
    int64_t rd = 0;
    for (int i = 0; i < a.g.size; ++i) {
      const int m = a.g.members[i];
      if (m / wpg != c->cfg.rank) continue;
      if (p.m >= rp::kMaxXLocal) return fail(RP_EINVAL, "more than 8 local members in a cross-GPU group");
      p.x[p.m] = c->w[m].x;
      p.u[p.m] = a.u[i];
      rd += member_bytes(a.u[i]) - 4;
      p.m++;
    }
    // HBM: reads (x, g, v) + v writes, partial write, the switch's read of this copy and
    // its write of the means, the owner's / copy-out stores of x, the copy-out reads
    hbm += rd * n + 4 * n + 8 * n + 4 * p.m * n + 4 * n * (p.kp - 1) / p.kp;
    nvl += 4 * n;  // per GPU and direction: ~4N for any kp
    c->stats.nvls_groups++;
    c->stats.groups_launched++;
    c->stats.cross_gpu_groups++;
  }
  const bool timing = (c->cfg.flags & RP_FLAG_TIMING) != 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timing) {
    e0 = timing_event(c);
    e1 = timing_event(c);
    if (!e0 || !e1) return fail(RP_ECUDA, "timing event creation failed");
    CUDA_TRY(cudaEventRecord(e0, stream));
  }
  std::string err;
  const int rc = rp::launch_nvls(T, stream, &err);
  if (rc != RP_OK) return fail(rc, err);
  if (timing) {
    CUDA_TRY(cudaEventRecord(e1, stream));
    c->timed.push_back({e0, e1, hbm, nvl, true, c->batches});
  }
  c->stats.kernel_launches++;
  c->stats.bytes_hbm += hbm;
  c->stats.bytes_nvlink += nvl;
  return RP_OK;
}

// Launch one asynchronous cross-GPU group on the comm stream (caller holds mu).
int launch_cross_async(rp_ctx* c, int64_t seq) {
  ActiveGroup& a = c->active.at(seq);
  c->stats.lock_assertions++;
  if (c->inflight & a.local_mask)
    return fail(RP_ECONFLICT, "atomicity violation: members " + members_str(a.g, c->inflight) +
                                  " hold an unfinished group");
  for (int m = 0; m < RP_MAX_WORLD; ++m)
    if ((a.local_mask >> m) & 1) CUDA_TRY(cudaStreamWaitEvent(c->comm, c->w[m].ev_arrive, 0));
  const int rc = nvls_group(c, a.g) ? launch_nvls_groups(c, {seq}, c->comm) : launch_cross(c, {seq}, c->comm);
  if (rc != RP_OK) return rc;
  WorkerSlot& L = c->w[__builtin_ctzll(a.local_mask)];
  CUDA_TRY(cudaEventRecord(L.ev_group, c->comm));
  for (int m = 0; m < RP_MAX_WORLD; ++m) {
    if (!((a.local_mask >> m) & 1)) continue;
    CUDA_TRY(cudaStreamWaitEvent(c->w[m].stream, L.ev_group, 0));
    CUDA_TRY(cudaEventRecord(c->w[m].ev_done, c->w[m].stream));
  }
  a.launched = true;
  c->inflight |= a.local_mask;
  c->cv.notify_all();
  return RP_OK;
}

// Launch asynchronous cross-GPU groups (shared GG). A group's parts are launched
// only once ALL its members, on every GPU, have arrived (no kernel ever spins on
// an absent member), and every GPU launches its parts in the order in which the
// groups became complete (the shared ticket). Two GPUs therefore never hold
// each other's later group behind an earlier one (the lowest ticket in flight
// can always finish), and a group waiting for a slow member delays nobody else.
// Caller holds mu. Waiting threads call it repeatedly (remote arrivals).
int pump_cross(rp_ctx* c) {
  const int wpg = c->cfg.workers_per_gpu;
  for (;;) {
    int64_t best = -1, best_ticket = -1;
    {
      GGLock gl(c);
      // lowest complete (ticketed) cross group involving this GPU not launched here yet
      for (const auto& g : c->ggp->table) {
        if (g.seq < 0 || g.ticket < 0 || c->xlaunched.count(g.seq)) continue;
        bool mine = false, other = false;
        for (int i = 0; i < g.size; ++i) (g.members[i] / wpg == c->cfg.rank ? mine : other) = true;
        if (!(mine && other)) continue;
        if (best_ticket < 0 || g.ticket < best_ticket) {
          best_ticket = g.ticket;
          best = g.seq;
        }
      }
    }
    // it must be launched before anything later; it is ours to launch once our local
    // members' arrival is recorded here (it always is: complete => every member arrived)
    if (best < 0 || !c->xready.count(best)) return RP_OK;
    c->xready.erase(best);
    c->xlaunched.insert(best);
    const int rc = launch_cross_async(c, best);
    if (rc != RP_OK) return rc;
  }
}

int open_shared_gg(rp_ctx* c) {
  const rp_config& k = c->cfg;
  // n_gpus == 0 (host-only) is allowed so the multi-process GG can be tested without GPUs
  if (k.n_gpus == 1 || k.job_id == 0) return fail(RP_EINVAL, "RP_FLAG_SHARED_GG needs n_gpus != 1 and a job_id");
  c->shm_name = "/rp_gg_" + std::to_string(static_cast<unsigned long long>(k.job_id));
  const size_t size = sizeof(SharedGG);
  int fd = -1;
  if (k.rank == 0) {
    shm_unlink(c->shm_name.c_str());
    fd = shm_open(c->shm_name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, static_cast<off_t>(size)) != 0) {
      if (fd >= 0) close(fd);
      return fail(RP_ENOMEM, "shared GG: cannot create " + c->shm_name);
    }
  } else {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      fd = shm_open(c->shm_name.c_str(), O_RDWR, 0600);
      struct stat st {};
      if (fd >= 0 && fstat(fd, &st) == 0 && static_cast<size_t>(st.st_size) >= size) break;
      if (fd >= 0) close(fd);
      fd = -1;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
        return fail(RP_ETIMEOUT, "shared GG: " + c->shm_name + " not created by rank 0");
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  void* p = mmap(nullptr, size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return fail(RP_ENOMEM, "shared GG: mmap failed");
  c->shm = static_cast<SharedGG*>(p);
  if (k.rank == 0) {
    pthread_mutexattr_t at;
    pthread_mutexattr_init(&at);
    pthread_mutexattr_setpshared(&at, PTHREAD_PROCESS_SHARED);
    pthread_mutex_init(&c->shm->mu, &at);
    pthread_mutexattr_destroy(&at);
    c->shm->trace_n = 0;
    rp::gg_init(&c->shm->gg, k.world, k.group_size, k.c_thres, k.seed_gd, c->gg.policy, c->gg.nodes);
    __atomic_store_n(&c->shm->magic, kSharedMagic, __ATOMIC_RELEASE);
  } else {
    const auto t0 = std::chrono::steady_clock::now();
    while (__atomic_load_n(&c->shm->magic, __ATOMIC_ACQUIRE) != kSharedMagic) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
        return fail(RP_ETIMEOUT, "shared GG: rank 0 never initialized " + c->shm_name);
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  c->ggp = &c->shm->gg;
  if (c->ggp->n != k.world || c->ggp->k != k.group_size)
    return fail(RP_EINVAL, "shared GG: configuration differs between ranks");
  return RP_OK;
}

using CuMemGetAddressRange = int (*)(uintptr_t*, size_t*, uintptr_t);

// Allocation base of a device pointer (driver entry point; no link-time libcuda).
int allocation_base(const void* p, uintptr_t* base) {
  static CuMemGetAddressRange fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
      return fail(RP_ECUDA, "cuMemGetAddressRange entry point unavailable");
    fn = reinterpret_cast<CuMemGetAddressRange>(f);
  }
  size_t size = 0;
  if (fn(base, &size, reinterpret_cast<uintptr_t>(p)) != 0) return fail(RP_ECUDA, "cuMemGetAddressRange failed");
  return RP_OK;
}

}  // namespace

extern "C" {

int rp_abi_version(void) { return RP_ABI_VERSION; }

const char* rp_last_error(void) { return rp::t_last_error.c_str(); }

const char* rp_strerror(int status) {
  switch (status) {
    case RP_OK: return "ok";
    case RP_EINVAL: return "invalid argument";
    case RP_ESTATE: return "invalid state";
    case RP_EPROTO: return "collective protocol error";
    case RP_ECONFLICT: return "conflicting groups (atomicity violation)";
    case RP_ETIMEOUT: return "timeout";
    case RP_ECUDA: return "CUDA error";
    case RP_ENOMEM: return "out of memory";
    case RP_ENODEV: return "no GPU in this context";
    case RP_EAGAIN: return "group pending (retry)";
    default: return "unknown status";
  }
}

namespace {
// Stream of the intra-GPU launch that runs beside a cross-GPU launch. RP_AUX_PRIO: 0 = default
// priority (default), 1 = higher than the cross launch's stream, -1 = lower (experiment knob).
cudaError_t create_aux_stream(cudaStream_t* s) {
  const char* v = std::getenv("RP_AUX_PRIO");
  const int want = v && *v ? std::atoi(v) : 0;
  if (want == 0) return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
  int least = 0, greatest = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
  if (e != cudaSuccess) return e;
  return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, want > 0 ? greatest : least);
}
}  // namespace

// Stream of the cross-GPU launch in split mode. RP_XS_PRIO=1 gives it the greatest priority,
// so its CTAs take SM slots ahead of retiring CTAs of the intra-GPU launch (with RP_DYN_TPC):
// steadier at N = 2, slower at N = 4 (profiles/r01_split/, profiles/r01_final3_4gpu/): off.
static cudaError_t create_cross_stream(cudaStream_t* s) {
  const char* v = std::getenv("RP_XS_PRIO");
  if (!(v && *v && std::atoi(v) == 1)) return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
  int least = 0, greatest = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
  if (e != cudaSuccess) return e;
  return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, greatest);
}

int rp_init(const rp_config* cfg, rp_ctx** out) {
  if (!cfg || !out) return fail(RP_EINVAL, "rp_init: null argument");
  *out = nullptr;
  const rp_config& k = *cfg;
  if (k.world < 1 || k.world > RP_MAX_WORLD) return fail(RP_EINVAL, "rp_init: world must be in [1, 64]");
  if (k.n_params <= 0) return fail(RP_EINVAL, "rp_init: n_params must be > 0");
  if (k.group_size < 1 || k.group_size > RP_MAX_GROUP || k.group_size > k.world)
    return fail(RP_EINVAL, "rp_init: group_size must be in [1, min(16, world)]");
  if (k.n_gpus < 0 || k.n_gpus > RP_MAX_GPUS) return fail(RP_EINVAL, "rp_init: n_gpus must be in [0, 8]");
  if (k.dtype != RP_DTYPE_F32 && k.dtype != RP_DTYPE_BF16) return fail(RP_EINVAL, "rp_init: unknown dtype");
  if (k.n_gpus > 0) {
    if (k.workers_per_gpu < 1 || k.n_gpus * k.workers_per_gpu != k.world)
      return fail(RP_EINVAL, "rp_init: world must equal n_gpus * workers_per_gpu");
    if (k.rank < 0 || k.rank >= k.n_gpus) return fail(RP_EINVAL, "rp_init: rank out of range");
  }
  if ((k.flags & RP_FLAG_EMULATE) && (k.n_gpus < 2 || k.rank != 0 || (k.flags & RP_FLAG_SHARED_GG)))
    return fail(RP_EINVAL, "rp_init: RP_FLAG_EMULATE needs n_gpus >= 2 virtual GPUs, rank 0 and a private GG");
  rp_ctx* c = new (std::nothrow) rp_ctx();
  if (!c) return fail(RP_ENOMEM, "rp_init: allocation failed");
  c->cfg = k;
  if (c->cfg.workers_per_gpu < 1) c->cfg.workers_per_gpu = k.world;
  const int policy = (k.flags & RP_FLAG_RANDOM_GG) ? rp::kPolicyRandom : rp::kPolicyGD;
  int ii_nodes = 0;
  if (k.flags & RP_FLAG_INTER_INTRA) {
    ii_nodes = k.nodes > 0 ? k.nodes : k.n_gpus;
    if (ii_nodes < 1 || k.world % ii_nodes != 0 || policy != rp::kPolicyGD) {
      delete c;
      return fail(RP_EINVAL, "rp_init: Inter-Intra needs world = nodes * m (cfg.nodes or n_gpus) and GD");
    }
  }
  rp::gg_init(&c->gg, k.world, k.group_size, k.c_thres, k.seed_gd, policy, ii_nodes);
  if (k.flags & RP_FLAG_SHARED_GG) {
    const int rc = open_shared_gg(c);
    if (rc != RP_OK) {
      rp_finalize(c);
      return rc;
    }
  }
  if (k.n_gpus > 0) {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
      delete c;
      return fail(RP_ENODEV, std::string("rp_init: no CUDA device: ") + cudaGetErrorString(e));
    }
    if (k.device < 0 || k.device >= ndev) {
      delete c;
      return fail(RP_EINVAL, "rp_init: device out of range");
    }
    e = cudaSetDevice(k.device);
    if (e != cudaSuccess) {
      delete c;
      return cuda_fail(e, "cudaSetDevice");
    }
    c->has_gpu = true;
    {  // once per process and device: load every kernel now, not at a first launch in a timed region
      static std::mutex pl_mu;
      static uint64_t pl_done = 0;
      std::lock_guard<std::mutex> pl(pl_mu);
      if (!((pl_done >> k.device) & 1)) {
        rp::preload_preduce();
        rp::preload_preduce_tma();
        if (k.n_gpus > 1) {
          rp::preload_xgpu_ws();
          rp::preload_xgpu();
        }
        cudaGetLastError();
        pl_done |= 1ull << k.device;
      }
    }
    c->emulate = (k.flags & RP_FLAG_EMULATE) != 0;
    const int wpg = c->cfg.workers_per_gpu;
    const int w_lo = c->emulate ? 0 : k.rank * wpg, w_hi = c->emulate ? k.world : (k.rank + 1) * wpg;
    for (int w = w_lo; w < w_hi; ++w) {
      WorkerSlot& s = c->w[w];
      s.local = true;
      if ((e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&s.ev_arrive, cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&s.ev_group, cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&s.ev_done, cudaEventDisableTiming)) != cudaSuccess) {
        rp_finalize(c);
        return cuda_fail(e, "rp_init: stream/event creation");
      }
      s.own_stream = true;
    }
    if (k.n_gpus > 1) {
      if ((e = cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking)) != cudaSuccess ||
          (e = create_aux_stream(&c->aux)) != cudaSuccess ||
          (e = create_cross_stream(&c->xs)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&c->ev_xjoin, cudaEventDisableTiming)) != cudaSuccess) {
        rp_finalize(c);
        return cuda_fail(e, "rp_init: comm streams");
      }
      if (const char* pp = std::getenv("RP_XGPU_PROFILE")) c->prof_path = pp;
      if (wpg > RP_MAX_LOCAL) {
        rp_finalize(c);
        return fail(RP_EINVAL, "rp_init: at most 16 workers per GPU in a multi-GPU job");
      }
      c->stage_region = (rp::xgpu_stage_region_bytes(k.n_params) + 255) / 256 * 256;
      // flag-wait watchdog: rp_config.watchdog_s (0 = default 600 s, < 0 = off), RP_WATCHDOG_S overrides
      double wd = k.watchdog_s == 0 ? 600.0 : (k.watchdog_s < 0 ? 0.0 : static_cast<double>(k.watchdog_s));
      if (const char* v = std::getenv("RP_WATCHDOG_S"))
        if (*v) wd = std::atof(v);
      c->watchdog_ns = wd > 0 ? static_cast<unsigned long long>(wd * 1e9) : 0ull;
      if ((e = cudaHostAlloc(reinterpret_cast<void**>(&c->xerr), sizeof(rp::XErr), cudaHostAllocMapped)) !=
              cudaSuccess ||
          (e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->xerr_dev), c->xerr, 0)) != cudaSuccess) {
        rp_finalize(c);
        return cuda_fail(e, "rp_init: watchdog record");
      }
      std::memset(c->xerr, 0, sizeof(rp::XErr));
      const int nflag = c->emulate ? k.n_gpus : 1;
      if ((e = cudaMalloc(&c->claim, sizeof(unsigned int) * rp::kXClaimWords * nflag)) != cudaSuccess ||
          (e = cudaMemset(c->claim, 0, sizeof(unsigned int) * rp::kXClaimWords * nflag)) != cudaSuccess) {
        rp_finalize(c);
        return cuda_fail(e, "rp_init: claim counters");
      }
      if ((e = cudaMalloc(&c->flags, rp::kFlagWords * 8 * nflag)) != cudaSuccess ||
          (e = cudaMemset(c->flags, 0, rp::kFlagWords * 8 * nflag)) != cudaSuccess ||
          (e = cudaMalloc(&c->stage, c->stage_region * wpg * nflag)) != cudaSuccess) {
        rp_finalize(c);
        return cuda_fail(e, "rp_init: flag buffers");
      }
      if (c->emulate) {  // virtual GPU d: flag array d, staging regions [d*wpg, (d+1)*wpg)
        c->vflags = c->flags;
        c->vstage = c->stage;
        if ((e = cudaMalloc(&c->d_tasks, sizeof(rp::XTask) * k.n_gpus)) != cudaSuccess) {
          rp_finalize(c);
          return cuda_fail(e, "rp_init: emulation task buffer");
        }
        c->peers_ready = true;
      }
    }
  }
  *out = c;
  return RP_OK;
}

int rp_peer_export(rp_ctx* c, rp_peer_info* out) {
  if (!c || !out) return fail(RP_EINVAL, "null argument");
  if (c->emulate) return fail(RP_ESTATE, "rp_peer_export: emulated GPUs share one process (RP_FLAG_EMULATE)");
  if (!c->has_gpu || c->cfg.n_gpus < 2 || !c->flags) return fail(RP_ESTATE, "rp_peer_export: not a multi-GPU context");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaSetDevice(c->cfg.device);
  std::memset(out, 0, sizeof(*out));
  const int wpg = c->cfg.workers_per_gpu;
  out->rank = c->cfg.rank;
  out->n_local = wpg;
  out->first_worker = c->cfg.rank * wpg;
  out->pid = static_cast<int32_t>(getpid());
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->flags));
  std::memcpy(out->flags_handle, &h, sizeof(h));
  out->flags_offset = 0;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->stage));
  std::memcpy(out->stage_handle, &h, sizeof(h));
  out->stage_offset = 0;
  out->stage_region_bytes = c->stage_region;
  for (int i = 0; i < wpg; ++i) {
    const WorkerSlot& s = c->w[out->first_worker + i];
    if (!s.bound) return fail(RP_ESTATE, "rp_peer_export: worker " + std::to_string(out->first_worker + i) + " not bound");
    uintptr_t base = 0;
    const int rc = allocation_base(s.x, &base);
    if (rc != RP_OK) return rc;
    CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(out->x_handle[i], &h, sizeof(h));
    out->x_offset[i] = static_cast<int64_t>(reinterpret_cast<uintptr_t>(s.x) - base);
  }
  return RP_OK;
}

int rp_peer_import(rp_ctx* c, const rp_peer_info* infos, int32_t n) {
  if (!c || !infos) return fail(RP_EINVAL, "null argument");
  if (c->emulate) return fail(RP_ESTATE, "rp_peer_import: emulated GPUs share one process (RP_FLAG_EMULATE)");
  if (!c->has_gpu || c->cfg.n_gpus < 2 || !c->flags) return fail(RP_ESTATE, "rp_peer_import: not a multi-GPU context");
  if (n != c->cfg.n_gpus) return fail(RP_EINVAL, "rp_peer_import: need one record per GPU");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaSetDevice(c->cfg.device);
  const int wpg = c->cfg.workers_per_gpu;
  bool seen[RP_MAX_GPUS] = {};
  // distinct allocations are opened once (several replicas may share one)
  std::vector<std::pair<std::string, void*>> opened;
  auto open = [&](const uint8_t* hb, void** out) -> int {
    const std::string key(reinterpret_cast<const char*>(hb), RP_IPC_HANDLE_BYTES);
    for (auto& kv : opened)
      if (kv.first == key) {
        *out = kv.second;
        return RP_OK;
      }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb, sizeof(h));
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    opened.emplace_back(key, p);
    c->ipc_mapped.push_back(p);
    *out = p;
    return RP_OK;
  };
  for (int i = 0; i < n; ++i) {
    const rp_peer_info& r = infos[i];
    if (r.rank < 0 || r.rank >= n || seen[r.rank] || r.n_local != wpg || r.first_worker != r.rank * wpg ||
        r.stage_region_bytes != c->stage_region)
      return fail(RP_EINVAL, "rp_peer_import: inconsistent record for rank " + std::to_string(r.rank));
    seen[r.rank] = true;
    c->peer_pid[r.rank] = r.pid;
    if (r.rank == c->cfg.rank) continue;
    void* fb = nullptr;
    int rc = open(r.flags_handle, &fb);
    if (rc != RP_OK) return rc;
    c->peer_flags[r.rank] = reinterpret_cast<unsigned long long*>(static_cast<char*>(fb) + r.flags_offset);
    void* sb = nullptr;
    rc = open(r.stage_handle, &sb);
    if (rc != RP_OK) return rc;
    c->peer_stage[r.rank] = reinterpret_cast<float*>(static_cast<char*>(sb) + r.stage_offset);
    for (int j = 0; j < wpg; ++j) {
      void* xb = nullptr;
      rc = open(r.x_handle[j], &xb);
      if (rc != RP_OK) return rc;
      c->peer_x[r.first_worker + j] = reinterpret_cast<float*>(static_cast<char*>(xb) + r.x_offset[j]);
    }
  }
  c->peers_ready = true;
  return RP_OK;
}

int rp_nvls_supported(rp_ctx* c, int32_t* supported) {
  if (!c || !supported) return fail(RP_EINVAL, "null argument");
  if (!c->has_gpu || c->cfg.n_gpus < 2) return fail(RP_ESTATE, "rp_nvls_supported: not a multi-GPU context");
  cudaSetDevice(c->cfg.device);
  int v = 0;
  rp::nvls_supported(c->cfg.device, &v);
  *supported = v;
  return RP_OK;
}

int rp_nvls_enable(rp_ctx* c, int32_t min_gpus, rp_barrier_fn barrier, void* user) {
  if (!c || !barrier) return fail(RP_EINVAL, "null argument");
  if (!c->has_gpu || c->cfg.n_gpus < 2) return fail(RP_ESTATE, "rp_nvls_enable: not a multi-GPU context");
  if (min_gpus < 2 || min_gpus > c->cfg.n_gpus) return fail(RP_EINVAL, "rp_nvls_enable: min_gpus out of range");
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->peers_ready) return fail(RP_ESTATE, "rp_nvls_enable: call rp_peer_import first");
  if (c->nvls.min_gpus > 0) return fail(RP_ESTATE, "rp_nvls_enable: already enabled");
  if (c->cfg.dtype != RP_DTYPE_F32) return fail(RP_EINVAL, "rp_nvls_enable: fp32 replicas only");
  int subsets = 0;
  for (uint32_t m = 1; m < (1u << c->cfg.n_gpus); ++m) subsets += __builtin_popcount(m) >= min_gpus;
  if (subsets > 64) return fail(RP_EINVAL, "rp_nvls_enable: more than 64 GPU subsets (P:1239 cache bound)");
  cudaSetDevice(c->cfg.device);
  std::string err;  // unsupported hardware fails inside, in step with the other ranks
  const int rc = rp::nvls_setup(&c->nvls, c->cfg.rank, c->cfg.n_gpus, c->cfg.device, c->cfg.workers_per_gpu,
                                c->cfg.n_params, min_gpus, c->peer_pid, barrier, user, &err);
  if (rc != RP_OK) return fail(rc, err);
  return RP_OK;
}

namespace {
void release_graph(const rp_ctx* c);
}

int rp_finalize(rp_ctx* c) {
  if (!c) return RP_OK;
  release_graph(c);
  if (c->has_gpu) {
    cudaSetDevice(c->cfg.device);
    for (auto& t : c->timed) {
      cudaEventDestroy(t.start);
      cudaEventDestroy(t.stop);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    if (c->comm) {
      cudaStreamSynchronize(c->comm);
      cudaStreamDestroy(c->comm);
    }
    if (c->aux) {
      cudaStreamSynchronize(c->aux);
      cudaStreamDestroy(c->aux);
    }
    if (c->xs) {
      cudaStreamSynchronize(c->xs);
      cudaStreamDestroy(c->xs);
    }
    cudaDeviceSynchronize();  // no kernel may still use the peer mappings closed below
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_xjoin) cudaEventDestroy(c->ev_xjoin);
    for (void* p : c->ipc_mapped) cudaIpcCloseMemHandle(p);
    cudaDeviceSynchronize();
    rp::nvls_teardown(&c->nvls);
    if (c->flags) cudaFree(c->flags);
    if (c->stage) cudaFree(c->stage);
    if (c->d_tasks) cudaFree(c->d_tasks);
    if (c->claim) cudaFree(c->claim);
    if (c->xerr) cudaFreeHost(c->xerr);
    if (c->prof) {
      // dump the item timeline of the last cross-GPU launch
      std::vector<rp::XItemRecord> h(c->prof_items);
      if (cudaMemcpy(h.data(), c->prof, h.size() * sizeof(rp::XItemRecord), cudaMemcpyDeviceToHost) == cudaSuccess) {
        const std::string path = c->prof_path + "." + std::to_string(c->cfg.rank);
        if (FILE* f = std::fopen(path.c_str(), "wb")) {
          std::fwrite(h.data(), sizeof(rp::XItemRecord), h.size(), f);
          std::fclose(f);
        }
      }
      cudaFree(c->prof);
    }
    if (c->cta_stat) {  // per-CTA breakdown [ring wait, signal wait, flag wait, total] ns of the last launch
      std::vector<unsigned long long> h(rp::kCtaStatWords);
      if (cudaMemcpy(h.data(), c->cta_stat, h.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
        const std::string path = c->prof_path + ".cta." + std::to_string(c->cfg.rank);
        if (FILE* f = std::fopen(path.c_str(), "wb")) {
          std::fwrite(h.data(), 8, h.size(), f);
          std::fclose(f);
        }
      }
      cudaFree(c->cta_stat);
    }
    for (auto& s : c->w) {
      if (s.stream) cudaStreamSynchronize(s.stream);
      if (s.ev_arrive) cudaEventDestroy(s.ev_arrive);
      if (s.ev_group) cudaEventDestroy(s.ev_group);
      if (s.ev_done) cudaEventDestroy(s.ev_done);
      if (s.own_stream && s.stream) cudaStreamDestroy(s.stream);
    }
  }
  if (c->trace) std::fclose(c->trace);
  if (c->shm) {
    munmap(c->shm, sizeof(SharedGG));
    if (c->cfg.rank == 0) shm_unlink(c->shm_name.c_str());
  }
  delete c;
  return RP_OK;
}

namespace {
int bind_worker(rp_ctx* c, int32_t w, float* x, const float* g);
}

int rp_bind_worker(rp_ctx* c, int32_t w, float* x, const float* g) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (c->cfg.dtype != RP_DTYPE_F32) return fail(RP_EINVAL, "rp_bind_worker: bf16 context (use rp_bind_worker_bf16)");
  return bind_worker(c, w, x, g);
}

int rp_bind_worker_bf16(rp_ctx* c, int32_t w, uint16_t* x, const uint16_t* g) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (c->cfg.dtype != RP_DTYPE_BF16) return fail(RP_EINVAL, "rp_bind_worker_bf16: fp32 context");
  return bind_worker(c, w, reinterpret_cast<float*>(x), reinterpret_cast<const float*>(g));
}

namespace {
int bind_worker(rp_ctx* c, int32_t w, float* x, const float* g) {
  if (!c->has_gpu) return fail(RP_ENODEV, "rp_bind_worker: host-only context");
  if (!worker_ok(c, w) || !c->w[w].local) return fail(RP_EINVAL, "rp_bind_worker: worker not local to this rank");
  if (!x || (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(g) & 15))
    return fail(RP_EINVAL, "rp_bind_worker: x (and g) must be non-null 16-byte aligned device pointers");
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, x) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
      pa.device != c->cfg.device) {
    cudaGetLastError();
    return fail(RP_EINVAL, "rp_bind_worker: x is not device memory of this rank's GPU");
  }
  std::lock_guard<std::mutex> lk(c->mu);
  c->w[w].x = x;
  c->w[w].g = g;
  c->w[w].bound = true;
  return RP_OK;
}
}  // namespace

int rp_worker_stream(rp_ctx* c, int32_t w, void** out) {
  if (!c || !out) return fail(RP_EINVAL, "null argument");
  if (!c->has_gpu) return fail(RP_ENODEV, "host-only context");
  if (!worker_ok(c, w) || !c->w[w].local) return fail(RP_EINVAL, "worker not local");
  *out = c->w[w].stream;
  return RP_OK;
}

int rp_set_worker_stream(rp_ctx* c, int32_t w, void* stream) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (!c->has_gpu) return fail(RP_ENODEV, "host-only context");
  if (!worker_ok(c, w) || !c->w[w].local) return fail(RP_EINVAL, "worker not local");
  std::lock_guard<std::mutex> lk(c->mu);
  WorkerSlot& s = c->w[w];
  if (s.in_group) return fail(RP_ESTATE, "worker is inside a group");
  cudaSetDevice(c->cfg.device);
  if (s.own_stream) {
    cudaStreamSynchronize(s.stream);
    cudaStreamDestroy(s.stream);
  }
  s.stream = static_cast<cudaStream_t>(stream);
  s.own_stream = false;
  return RP_OK;
}

int rp_schedule_static(rp_ctx* c, int32_t rule, int64_t step, int32_t* group_of, int32_t* n_groups) {
  if (!c || !group_of || !n_groups) return fail(RP_EINVAL, "null argument");
  if (rule == RP_SCHED_PAPER4) {
    const int nodes = c->cfg.nodes > 0 ? c->cfg.nodes : c->cfg.n_gpus;
    if (nodes < 1 || c->cfg.world % nodes != 0)
      return fail(RP_EINVAL, "PAPER4 needs world = nodes * m (set cfg.nodes)");
    return rp::schedule_paper4(nodes, c->cfg.world / nodes, step, group_of, n_groups);
  }
  if (rule == RP_SCHED_SHIFT_K) return rp::schedule_shift_k(c->cfg.world, c->cfg.group_size, step, group_of, n_groups);
  return fail(RP_EINVAL, "unknown schedule rule");
}

int rp_schedule_static_worker(rp_ctx* c, int32_t rule, int64_t step, int32_t w, rp_group* out) {
  if (!c || !out) return fail(RP_EINVAL, "null argument");
  if (!worker_ok(c, w)) return fail(RP_EINVAL, "worker out of range");
  int32_t group_of[RP_MAX_WORLD];
  int32_t ng = 0;
  const int rc = rp_schedule_static(c, rule, step, group_of, &ng);
  if (rc != RP_OK) return rc;
  std::memset(out, 0xff, sizeof(*out));
  out->size = 0;
  if (group_of[w] < 0) {
    out->members[out->size++] = w;
  } else {
    for (int v = 0; v < c->cfg.world; ++v)
      if (group_of[v] == group_of[w]) {
        if (out->size >= RP_MAX_GROUP) return fail(RP_EINVAL, "static group larger than RP_MAX_GROUP");
        out->members[out->size++] = v;
      }
  }
  out->seq = -(1 + step * c->cfg.world + out->members[0]);
  return RP_OK;
}

int rp_group_generate(rp_ctx* c, int32_t w, rp_group* out) {
  if (!c || !out) return fail(RP_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  GGLock gl(c);
  const int rc = rp::gg_request(c->ggp, w, out);
  if (rc == RP_EAGAIN) {
    trace_line(c, "\"ev\":\"req\",\"w\":" + std::to_string(w) + ",\"pending\":" + std::to_string(out->seq));
    return fail(RP_EAGAIN, "group " + std::to_string(out->seq) + " of worker " + std::to_string(w) +
                               " waits in the pending queue");
  }
  if (rc != RP_OK) return rc;
  c->stats.gg_requests++;
  trace_line(c, "\"ev\":\"req\",\"w\":" + std::to_string(w) + "," + group_json(*out));
  return RP_OK;
}

int rp_group_generate_many(rp_ctx* c, const int32_t* workers, int32_t n, rp_group* out) {
  if (!c || (n > 0 && (!workers || !out)) || n < 0) return fail(RP_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lk(c->mu);
  GGLock gl(c);
  for (int i = 0; i < n; ++i) {
    const int rc = rp::gg_request(c->ggp, workers[i], &out[i]);
    if (rc != RP_OK) return rc;
    c->stats.gg_requests++;
    trace_line(c, "\"ev\":\"req\",\"w\":" + std::to_string(workers[i]) + "," + group_json(out[i]));
  }
  return RP_OK;
}

int rp_gg_release(rp_ctx* c, int64_t seq) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  std::lock_guard<std::mutex> lk(c->mu);
  if (c->active.count(seq)) return fail(RP_ESTATE, "rp_gg_release: group is executed by this process");
  return release_gg_group(c, seq);
}

int rp_retire(rp_ctx* c, int32_t w) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  std::lock_guard<std::mutex> lk(c->mu);
  GGLock gl(c);
  const int rc = rp::gg_retire(c->ggp, w);
  if (rc == RP_OK) trace_line(c, "\"ev\":\"retire\",\"w\":" + std::to_string(w));
  return rc;
}

namespace {
int stage_step(rp_ctx* c, int32_t w, const float* grad, float lr);
}

int rp_step(rp_ctx* c, int32_t w, const float* grad, float lr) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (c->cfg.dtype != RP_DTYPE_F32 && grad)
    return fail(RP_EINVAL, "rp_step: bf16 context takes a bf16 gradient (rp_step_bf16)");
  return stage_step(c, w, grad, lr);
}

int rp_step_bf16(rp_ctx* c, int32_t w, const uint16_t* grad, float lr) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (c->cfg.dtype != RP_DTYPE_BF16) return fail(RP_EINVAL, "rp_step_bf16: fp32 context");
  return stage_step(c, w, reinterpret_cast<const float*>(grad), lr);
}

namespace {
int stage_step(rp_ctx* c, int32_t w, const float* grad, float lr) {
  if (!c->has_gpu) return fail(RP_ENODEV, "rp_step: host-only context");
  if (!worker_ok(c, w) || !c->w[w].local) return fail(RP_EINVAL, "rp_step: worker not local");
  std::lock_guard<std::mutex> lk(c->mu);
  WorkerSlot& s = c->w[w];
  if (!s.bound) return fail(RP_ESTATE, "rp_step: worker not bound");
  if (s.staged) return fail(RP_ESTATE, "rp_step: a step is already staged for worker " + std::to_string(w));
  const float* gp = grad ? grad : s.g;
  if (!gp) return fail(RP_EINVAL, "rp_step: no gradient buffer");
  if (reinterpret_cast<uintptr_t>(gp) & 15) return fail(RP_EINVAL, "rp_step: gradient must be 16-byte aligned");
  s.staged = true;
  s.upd = rp::MemberUpdate{gp, nullptr, lr, 0.f, 0.f};
  return RP_OK;
}
}  // namespace

int rp_step_momentum(rp_ctx* c, int32_t w, const float* grad, float lr, float momentum, float weight_decay,
                     float* v_dev) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (c->cfg.dtype != RP_DTYPE_F32) return fail(RP_EINVAL, "rp_step_momentum: fp32 replicas only");
  if (!v_dev || (reinterpret_cast<uintptr_t>(v_dev) & 15))
    return fail(RP_EINVAL, "rp_step_momentum: momentum buffer must be a non-null 16-byte aligned device pointer");
  const int rc = rp_step(c, w, grad, lr);
  if (rc != RP_OK) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  WorkerSlot& s = c->w[w];
  s.upd.v = v_dev;
  s.upd.mu = momentum;
  s.upd.wd = weight_decay;
  return RP_OK;
}

int rp_preduce(rp_ctx* c, int32_t w, const rp_group* g) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (!c->has_gpu) return fail(RP_ENODEV, "rp_preduce: host-only context");
  if (!worker_ok(c, w) || !c->w[w].local) return fail(RP_EINVAL, "rp_preduce: worker not local");
  uint64_t mask = 0;
  int rc = check_group(c, g, &mask);
  if (rc != RP_OK) return rc;
  if (!((mask >> w) & 1)) return fail(RP_EPROTO, "rp_preduce: worker " + std::to_string(w) + " not in group");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaSetDevice(c->cfg.device);
  WorkerSlot& s = c->w[w];
  if (!s.bound) return fail(RP_ESTATE, "rp_preduce: worker not bound");
  if (s.in_group)
    return fail(RP_ESTATE, "rp_preduce: worker " + std::to_string(w) + " has not waited for group " +
                               std::to_string(s.seq));
  if (g->seq >= 0) {  // GG group: must be the one handed to w
    GGLock gl(c);
    rp::GGGroup* gg = const_cast<rp::GGGroup*>(rp::gg_find(c->ggp, g->seq));
    bool ok = gg && c->ggp->handed[w] == g->seq && gg->size == g->size;
    for (int i = 0; ok && i < g->size; ++i) ok = gg->members[i] == g->members[i];
    if (ok && c->shm) {  // global arrival record; the completing arrival takes the next ticket
      gg->arrived |= 1ull << w;
      if (gg->ticket < 0 && gg->arrived == mask) gg->ticket = c->ggp->next_ticket++;
    }
    if (!ok) return fail(RP_EPROTO, "rp_preduce: group " + std::to_string(g->seq) + " was not handed to worker " +
                                        std::to_string(w) + " by the GG");
  }
  auto it = c->active.find(g->seq);
  if (it == c->active.end()) {
    ActiveGroup a;
    a.g = *g;
    a.members_mask = mask;
    const int wpg = c->cfg.workers_per_gpu;
    for (int i = 0; i < g->size; ++i)
      if (c->emulate || g->members[i] / wpg == c->cfg.rank) a.local_mask |= 1ull << g->members[i];
    it = c->active.emplace(g->seq, a).first;
  } else if (!same_group(it->second.g, *g)) {
    return fail(RP_EPROTO, "rp_preduce: members disagree on group " + std::to_string(g->seq) + ": " +
                               members_str(it->second.g) + " vs " + members_str(*g));
  }
  ActiveGroup& a = it->second;
  if ((a.arrived >> w) & 1) return fail(RP_EPROTO, "rp_preduce: worker arrived twice");
  if (is_cross(c, a) && !c->batching && !(c->shm && g->seq >= 0 && !c->emulate))
    return fail(RP_ESTATE, "rp_preduce: a cross-GPU group must be issued inside rp_batch_begin/end "
                           "(one launch per GPU and step keeps the GPUs' launch orders consistent), "
                           "or be a shared-GG group (RP_FLAG_SHARED_GG)");
  int idx = 0;
  while (g->members[idx] != w) ++idx;
  a.u[idx] = s.staged ? s.upd : rp::MemberUpdate{};
  CUDA_TRY(cudaEventRecord(s.ev_arrive, s.stream));
  s.staged = false;
  s.in_group = true;
  s.seq = g->seq;
  a.arrived |= 1ull << w;
  if ((a.arrived & a.local_mask) == a.local_mask) {
    if (c->batching) {
      c->ready.push_back(g->seq);
      return RP_OK;
    }
    if (a.local_mask != a.members_mask) {  // asynchronous cross-GPU group: GG order
      c->xready.insert(g->seq);
      return pump_cross(c);
    }
    return launch_groups(c, {g->seq});
  }
  return RP_OK;
}

int rp_barrier_free_wait(rp_ctx* c, int32_t w, int64_t timeout_us) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (!c->has_gpu) return fail(RP_ENODEV, "host-only context");
  if (!worker_ok(c, w) || !c->w[w].local) return fail(RP_EINVAL, "worker not local");
  const auto t0 = std::chrono::steady_clock::now();
  const auto deadline = t0 + std::chrono::microseconds(timeout_us < 0 ? 0 : timeout_us);
  std::unique_lock<std::mutex> lk(c->mu);
  WorkerSlot& s = c->w[w];
  if (!s.in_group) return fail(RP_ESTATE, "rp_barrier_free_wait: worker " + std::to_string(w) + " is not in a group");
  const int64_t seq = s.seq;
  auto missing = [&](const ActiveGroup& a) { return members_str(a.g, a.members_mask & ~a.arrived); };
  {
    ActiveGroup& a = c->active.at(seq);
    if (!a.launched) {
      if (timeout_us < 0)
        return fail(RP_ESTATE, "group " + std::to_string(seq) + " not launched; missing members " + missing(a));
      for (;;) {
        if (c->shm) {  // remote members arrive in other processes: drive the launcher here
          const int prc = pump_cross(c);
          if (prc != RP_OK) return prc;
        }
        if (c->active.at(seq).launched) break;
        if (std::chrono::steady_clock::now() >= deadline)
          return fail(RP_ETIMEOUT, "group " + std::to_string(seq) + " " + members_str(a.g) +
                                       ": members never arrived: " + missing(c->active.at(seq)));
        c->cv.wait_for(lk, std::chrono::microseconds(c->shm ? 20 : 1000));
      }
    }
  }
  if (timeout_us >= 0) {
    cudaEvent_t ev = s.ev_done;
    lk.unlock();
    cudaSetDevice(c->cfg.device);
    for (;;) {
      const cudaError_t e = cudaEventQuery(ev);
      if (e == cudaSuccess) break;
      if (e != cudaErrorNotReady) return cuda_fail(e, "cudaEventQuery");
      if (std::chrono::steady_clock::now() >= deadline)
        return fail(RP_ETIMEOUT, "group " + std::to_string(seq) + " launched but not complete");
      std::this_thread::yield();
    }
    lk.lock();
    const int xrc = check_xerr(c);
    if (xrc != RP_OK) return xrc;
  }
  ActiveGroup& a = c->active.at(seq);
  s.in_group = false;
  c->inflight &= ~(1ull << w);
  a.waited |= 1ull << w;
  // Reading R11: the GG releases the group at the first observation of its
  // completion (host-observed, or stream-ordered for RP_WAIT_DEVICE), so the
  // members' Group Buffers advance even if some member has not waited yet.
  int rc = RP_OK;
  if (!a.released) {
    a.released = true;
    if (seq >= 0) rc = release_gg_group(c, seq);
  }
  if ((a.waited & a.local_mask) == a.local_mask) {
    c->active.erase(seq);
    c->xlaunched.erase(seq);
  }
  return rc;
}

int rp_batch_begin(rp_ctx* c) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (!c->has_gpu) return fail(RP_ENODEV, "host-only context");
  std::lock_guard<std::mutex> lk(c->mu);
  if (c->batching) return fail(RP_ESTATE, "rp_batch_begin: already batching");
  c->batching = true;
  return RP_OK;
}

int rp_batch_end(rp_ctx* c) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (!c->has_gpu) return fail(RP_ENODEV, "host-only context");
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->batching) return fail(RP_ESTATE, "rp_batch_end: no batch open");
  c->batching = false;
  cudaSetDevice(c->cfg.device);
  std::vector<int64_t> q;
  q.swap(c->ready);
  const int rc = launch_groups(c, q);
  c->batches++;
  return rc;
}

int rp_set_compute_delay(rp_ctx* c, int32_t w, int64_t ns) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (!c->has_gpu) return fail(RP_ENODEV, "host-only context");
  if (!worker_ok(c, w) || !c->w[w].local || ns < 0) return fail(RP_EINVAL, "rp_set_compute_delay: bad worker or ns");
  std::lock_guard<std::mutex> lk(c->mu);
  c->w[w].delay_ns = ns;
  return RP_OK;
}

int rp_check(rp_ctx* c) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  return check_xerr(c);
}

int rp_timing_read(rp_ctx* c, rp_timing* out) {
  if (!c || !out) return fail(RP_EINVAL, "null argument");
  if (!(c->cfg.flags & RP_FLAG_TIMING)) return fail(RP_ESTATE, "context created without RP_FLAG_TIMING");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaSetDevice(c->cfg.device);
  rp_timing r{};
  r.min_ms = 0;
  for (auto& t : c->timed) {
    CUDA_TRY(cudaEventSynchronize(t.stop));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, t.start, t.stop));
    r.launches++;
    r.total_ms += ms;
    r.min_ms = r.launches == 1 ? ms : std::min<double>(r.min_ms, ms);
    r.max_ms = std::max<double>(r.max_ms, ms);
    r.bytes_hbm += t.bytes_hbm;
    r.bytes_nvlink += t.bytes_nvlink;
    if (t.cross) {
      r.cross_launches++;
      r.cross_ms += ms;
      r.cross_bytes_nvlink += t.bytes_nvlink;
      r.cross_bytes_hbm += t.bytes_hbm;
    } else {
      r.local_launches++;
      r.local_ms += ms;
      r.local_bytes_hbm += t.bytes_hbm;
    }
    c->event_pool.push_back(t.start);
    c->event_pool.push_back(t.stop);
  }
  c->timed.clear();
  *out = r;
  return RP_OK;
}

int rp_timing_records(rp_ctx* c, rp_launch_record* out, int32_t cap, int32_t* n) {
  if (!c || !n || cap < 0 || (cap > 0 && !out)) return fail(RP_EINVAL, "bad argument");
  if (!(c->cfg.flags & RP_FLAG_TIMING)) return fail(RP_ESTATE, "context created without RP_FLAG_TIMING");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaSetDevice(c->cfg.device);
  const size_t k = std::min<size_t>(static_cast<size_t>(cap), c->timed.size());
  for (size_t i = 0; i < k; ++i) {
    auto& t = c->timed[i];
    CUDA_TRY(cudaEventSynchronize(t.stop));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, t.start, t.stop));
    out[i] = rp_launch_record{ms, t.bytes_hbm, t.bytes_nvlink, t.batch, t.cross ? 1 : 0, 0};
    c->event_pool.push_back(t.start);
    c->event_pool.push_back(t.stop);
  }
  c->timed.erase(c->timed.begin(), c->timed.begin() + static_cast<std::ptrdiff_t>(k));
  *n = static_cast<int32_t>(k);
  return RP_OK;
}

int rp_stats_get(rp_ctx* c, rp_stats* out) {
  if (!c || !out) return fail(RP_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  *out = c->stats;
  GGLock gl(c);
  out->gd_calls = c->ggp->gd_calls;
  out->max_gb_depth = c->ggp->max_depth;
  out->gg_pending = c->ggp->n_pending;
  out->gg_granted = c->ggp->n_granted;
  return RP_OK;
}

int rp_trace_open(rp_ctx* c, const char* path) {
  if (!c || !path) return fail(RP_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  if (c->trace) std::fclose(c->trace);
  c->trace = std::fopen(path, "w");
  if (!c->trace) return fail(RP_EINVAL, std::string("cannot open trace file ") + path);
  return RP_OK;
}

int rp_compute_delay(void* stream, int64_t ns) {
  std::string err;
  const int rc = rp::launch_delay(stream, ns, &err);
  return rc == RP_OK ? rc : fail(rc, err);
}

int rp_fill_xi(float* dst, int64_t n, uint64_t seed, uint64_t w, uint64_t t, uint64_t j0, void* stream) {
  std::string err;
  const int rc = rp::launch_fill_xi(dst, n, seed, w, t, j0, stream, &err);
  return rc == RP_OK ? rc : fail(rc, err);
}

}  // extern "C"

// Native lockstep executor: the LockstepRunner's step loop (runner.py) composed from the public
// calls above, so a lockstep step costs no per-call host overhead beyond C++.
namespace {
int lockstep_steps(rp_ctx* c, int32_t rule, int64_t t0, int64_t steps, float lr, int32_t section_length);
int lockstep_graph(rp_ctx* c, int32_t rule, int64_t t0, int64_t steps, float lr, int32_t section_length);
}  // namespace

int rp_lockstep_run(rp_ctx* c, int32_t rule, int64_t t0, int64_t steps, float lr, int32_t section_length) {
  if (!c) return fail(RP_EINVAL, "null ctx");
  if (!c->has_gpu) return fail(RP_ENODEV, "rp_lockstep_run: host-only context");
  if (steps < 0 || t0 < 1 || section_length < 1 ||
      (rule != RP_SCHED_GG && rule != RP_SCHED_PAPER4 && rule != RP_SCHED_SHIFT_K))
    return fail(RP_EINVAL, "rp_lockstep_run: bad rule, t0, steps or section_length");
  bool delays = false;
  for (int w = 0; w < c->cfg.world; ++w) delays = delays || (c->w[w].local && c->w[w].delay_ns > 0);
  if ((c->cfg.flags & RP_FLAG_GRAPH) && rule != RP_SCHED_GG && c->cfg.n_gpus <= 1 && !delays)
    return lockstep_graph(c, rule, t0, steps, lr, section_length);
  return lockstep_steps(c, rule, t0, steps, lr, section_length);
}

namespace {

// RP_FLAG_GRAPH: a static schedule repeats with period lcm(P, L) (P = 4 for PAPER4, k for SHIFT_K;
// L = section length), and so does every launch of one period (kernel arguments do not depend
// on t). One period of the native step loop is captured once into a CUDA graph (every worker
// stream joins the capture, so the group-local event ordering is kept as graph edges) and
// replayed; the remaining steps run through the plain loop. Host bookkeeping of a period is
// identical every time (all groups complete within their step), so the stats are advanced by
// the captured period's deltas. Timing events are not captured (RP_FLAG_TIMING is ignored
// inside the graph).
struct GraphCache {
  int32_t rule = 0, section = 0;
  int64_t phase = -1, period = 0;
  uint32_t lr_bits = 0;
  cudaGraphExec_t exec = nullptr;
  rp_stats delta{};
};
std::mutex g_graph_mu;
std::map<const rp_ctx*, GraphCache> g_graphs;

int64_t gcd64(int64_t a, int64_t b) { return b ? gcd64(b, a % b) : a; }

void add_stats(rp_stats& a, const rp_stats& d, int64_t times) {
  a.groups_launched += d.groups_launched * times;
  a.singleton_groups += d.singleton_groups * times;
  a.cross_gpu_groups += d.cross_gpu_groups * times;
  a.kernel_launches += d.kernel_launches * times;
  a.lock_assertions += d.lock_assertions * times;
  a.bytes_hbm += d.bytes_hbm * times;
  a.bytes_nvlink += d.bytes_nvlink * times;
}

int lockstep_graph(rp_ctx* c, int32_t rule, int64_t t0, int64_t steps, float lr, int32_t section_length) {
  const int64_t P = rule == RP_SCHED_PAPER4 ? 4 : std::max(1, c->cfg.group_size);
  const int64_t period = P / gcd64(P, section_length) * section_length;
  if (steps < period) return lockstep_steps(c, rule, t0, steps, lr, section_length);
  std::vector<int32_t> local;
  for (int w = 0; w < c->cfg.world; ++w)
    if (c->w[w].local) local.push_back(w);
  cudaStream_t s0 = c->w[local[0]].stream;
  uint32_t lr_bits = 0;
  std::memcpy(&lr_bits, &lr, 4);
  std::lock_guard<std::mutex> glk(g_graph_mu);
  GraphCache& G = g_graphs[c];
  if (!G.exec || G.rule != rule || G.section != section_length || G.phase != t0 % period || G.lr_bits != lr_bits) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    G = GraphCache{};
    cudaSetDevice(c->cfg.device);
    CUDA_TRY(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
    // every other worker stream joins the capture through an event recorded on s0
    int rc = RP_OK;
    cudaError_t e = cudaEventRecord(c->w[local[0]].ev_group, s0);
    for (size_t i = 1; i < local.size() && e == cudaSuccess; ++i)
      e = cudaStreamWaitEvent(c->w[local[i]].stream, c->w[local[0]].ev_group, 0);
    const rp_stats before = c->stats;
    const int32_t saved = c->cfg.flags;
    if (e == cudaSuccess) {
      c->cfg.flags &= ~RP_FLAG_TIMING;
      rc = lockstep_steps(c, rule, t0, period, lr, section_length);
      c->cfg.flags = saved;
    }
    // ... and joins back: s0 waits for the last event of every other worker stream
    for (size_t i = 1; i < local.size() && e == cudaSuccess; ++i) {
      e = cudaEventRecord(c->w[local[i]].ev_done, c->w[local[i]].stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s0, c->w[local[i]].ev_done, 0);
    }
    cudaGraph_t graph = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(s0, &graph);
    if (e != cudaSuccess) return cuda_fail(e, "rp_lockstep_run: graph capture");
    if (e2 != cudaSuccess) return cuda_fail(e2, "cudaStreamEndCapture");
    if (rc != RP_OK) {
      cudaGraphDestroy(graph);
      return rc;
    }
    e = cudaGraphInstantiate(&G.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    G.rule = rule;
    G.section = section_length;
    G.phase = t0 % period;
    G.period = period;
    G.lr_bits = lr_bits;
    G.delta = rp_stats{};
    rp_stats d = c->stats;  // the capture advanced the host counters by one period
    d.groups_launched -= before.groups_launched;
    d.singleton_groups -= before.singleton_groups;
    d.cross_gpu_groups -= before.cross_gpu_groups;
    d.kernel_launches -= before.kernel_launches;
    d.lock_assertions -= before.lock_assertions;
    d.bytes_hbm -= before.bytes_hbm;
    d.bytes_nvlink -= before.bytes_nvlink;
    G.delta = d;
    add_stats(c->stats, d, -1);  // counted again per replay below
  }
  const int64_t reps = steps / period;
  for (int64_t r = 0; r < reps; ++r) CUDA_TRY(cudaGraphLaunch(G.exec, s0));
  {
    std::lock_guard<std::mutex> lk(c->mu);
    add_stats(c->stats, G.delta, reps);
  }
  // later work on any worker stream is ordered after the replays
  CUDA_TRY(cudaEventRecord(c->w[local[0]].ev_group, s0));
  for (size_t i = 1; i < local.size(); ++i)
    CUDA_TRY(cudaStreamWaitEvent(c->w[local[i]].stream, c->w[local[0]].ev_group, 0));
  const int64_t rest = steps - reps * period;
  return rest ? lockstep_steps(c, rule, t0 + reps * period, rest, lr, section_length) : RP_OK;
}

int lockstep_steps(rp_ctx* c, int32_t rule, int64_t t0, int64_t steps, float lr, int32_t section_length) {
  const int world = c->cfg.world;
  std::vector<int32_t> local, all(world);
  std::vector<char> is_local(world, 0);
  for (int w = 0; w < world; ++w) {
    all[w] = w;
    if (c->w[w].local) {
      local.push_back(w);
      is_local[w] = 1;
    }
  }
  std::vector<rp_group> mine(local.size()), gen(world);
  std::vector<int64_t> foreign;
  for (int64_t s = 0; s < steps; ++s) {
    const int64_t t = t0 + s;
    const int xrc = check_xerr(c);  // a cross-GPU wait of an earlier (completed) launch gave up
    if (xrc != RP_OK) return xrc;
    for (int32_t w : local) {  // synthetic compute (harness), then alg1 step 2 with the bound gradient
      if (c->w[w].delay_ns > 0) {
        std::string err;
        const int drc = rp::launch_delay(c->w[w].stream, c->w[w].delay_ns, &err);
        if (drc != RP_OK) return fail(drc, err);
      }
      const int rc = stage_step(c, w, nullptr, lr);
      if (rc != RP_OK) return rc;
    }
    foreign.clear();
    if (t % section_length != 0) {  // no synchronization this step, SGD only
      for (size_t i = 0; i < local.size(); ++i) {
        mine[i] = rp_group{};
        mine[i].seq = -(1 + t * world + local[i]);
        mine[i].size = 1;
        for (int j = 0; j < RP_MAX_GROUP; ++j) mine[i].members[j] = j == 0 ? local[i] : -1;
      }
    } else if (rule != RP_SCHED_GG) {  // static schedule S(rule, t)
      for (size_t i = 0; i < local.size(); ++i) {
        const int rc = rp_schedule_static_worker(c, rule, t, local[i], &mine[i]);
        if (rc != RP_OK) return rc;
      }
    } else {  // GG requests of every worker in ascending order: identical on every rank
      int rc = rp_group_generate_many(c, all.data(), world, gen.data());
      if (rc != RP_OK) return rc;
      std::set<int64_t> seen;
      size_t li = 0;
      for (int w = 0; w < world; ++w) {
        const rp_group& g = gen[w];
        if (is_local[w]) {
          mine[li++] = g;
        } else if (!seen.count(g.seq)) {
          bool any_local = false;
          for (int j = 0; j < g.size; ++j) any_local = any_local || is_local[g.members[j]];
          if (!any_local) foreign.push_back(g.seq);
        }
        seen.insert(g.seq);
      }
    }
    int rc = rp_batch_begin(c);
    if (rc != RP_OK) return rc;
    for (size_t i = 0; i < local.size() && rc == RP_OK; ++i) rc = rp_preduce(c, local[i], &mine[i]);
    const int rc_end = rp_batch_end(c);
    if (rc != RP_OK) return rc;
    if (rc_end != RP_OK) return rc_end;
    for (int32_t w : local) {
      rc = rp_barrier_free_wait(c, w, RP_WAIT_DEVICE);
      if (rc != RP_OK) return rc;
    }
    std::sort(foreign.begin(), foreign.end());
    foreign.erase(std::unique(foreign.begin(), foreign.end()), foreign.end());
    for (int64_t q : foreign) {
      rc = rp_gg_release(c, q);
      if (rc != RP_OK) return rc;
    }
  }
  return RP_OK;
}

void release_graph(const rp_ctx* c) {
  std::lock_guard<std::mutex> glk(g_graph_mu);
  auto it = g_graphs.find(c);
  if (it == g_graphs.end()) return;
  if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
  g_graphs.erase(it);
}

}  // namespace
