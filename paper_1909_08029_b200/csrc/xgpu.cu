// Cross-GPU fused SGD + P-Reduce: this GPU's part of groups whose members span several GPUs
// of one NVSwitch node (one process per GPU, peer memory mapped through CUDA IPC), or all
// GPUs' parts emulated by one cooperative launch on a single device (RP_FLAG_EMULATE).
//
// alg1 step 4 for a group G on GPUs d_0 < ... < d_{kp-1} is one exchange step: a
// reduce-scatter + all-gather fused with the SGD of step 2 and with the pre-reduction of
// co-resident members (reading R1). The element range is cut into kp owner slices (GPU d_i owns
// slice i) and every slice into nch chunks. For one chunk index c this GPU runs, in order:
//
//  A(c)  for every owner o != me: p = left fold over my local members of y_m = fl(x_m - fl(lr_m g_m))
//        (ascending worker id) over chunk c of slice o, staged in shared memory tile by tile and
//        pushed by TMA bulk stores (cp.async.bulk global <- shared::cta) OVER NVLINK into owner
//        o's staging buffer (row me); then flag A[me][c] on o.
//  B(c)  my slice: wait for A[d][c] from every peer d; own partial in registers, the peers' from
//        my staging (local HBM); s = left fold of the partials in ascending GPU id; xbar =
//        fl(s / |G|) (reading R1); store xbar into my local members and push it (bulk stores,
//        OVER NVLINK) into every peer's first local member; then flag B[me][c] on every peer.
//  C(c)  for every owner o != me: wait for B[o][c]; copy xbar from my first local member to my
//        other local members (nothing to copy for a lone member, but the wait stays: a GPU
//        leaves the kernel only after every peer's last store into its memory).
//
// Schedule ("lanes"): chunk c belongs to lane c mod kXLanes. A CTA runs a lane as a software
// pipeline, iteration i = { A(c_i), B(c_{i-1}), C(c_{i-2}), signal }, so its NVLink pushes of
// chunk c_i travel while it folds chunk c_{i-1}: there is no phase barrier, every CTA carries the
// same mix of reduce-scatter and all-gather work, and one wait for its bulk stores per iteration publishes
// all of its flags (round 1 ran every A item before any B item; B items, one per chunk of the
// slice, left a third of the CTAs idle: profiles/r01_xall/timeline_n4.txt). The chunk geometry
// depends on (n, kp) only, never on the grid or the instantiation, so every GPU of a group cuts
// the same chunks whatever grid it launched. Lanes are taken in one global order (lane-major,
// then part) by every GPU and A never waits on B or C, so CTAs that spin on flags cannot form a
// cycle.
//
// NVLink bytes stored per GPU per group: A (kp-1)/kp * 4N + B (kp-1) * 4N/kp = 2 (kp-1)/kp * 4N,
// the ring all-reduce bus bound; no GPU reads peer memory (bidirectional peer stores 700 GB/s per
// direction vs 662 for loads, profiles/r01_nvlink_probe_2gpu.txt).
//
// Synchronization: 64-bit tags, unique per (group launch, GPU pair), in per-GPU flag arrays,
// published with st.release.sys after the bulk stores completed (cp.async.bulk.wait_group 0,
// fence.proxy.async) and polled with ld.acquire.sys. At kernel start each GPU
// posts READY to its peers; pushes into an owner's staging wait for its READY (its previous
// kernel, which read that staging, has finished). A flag wait longer than the watchdog limit
// (rp_config.watchdog_s / RP_WATCHDOG_S) records the flag in host-mapped memory and ends the
// CTA; the host reports RP_ETIMEOUT (no __trap, the context stays usable for diagnosis).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "rp_internal.h"
#include "update.cuh"

namespace rp {

namespace {

#ifndef RP_XGPU_MINB
#define RP_XGPU_MINB 2  // resident CTAs per SM the register allocation targets
#endif
constexpr int kXThreads = 256;
constexpr int kRowF4 = kXThreads;                 // vectors per tile row (one per thread)
constexpr int kTileRows = 4;
constexpr int64_t kTileF4 = kRowF4 * kTileRows;   // 1024 vectors: a 16 KB fp32 tile
constexpr int kNbufDefault = 3;                   // shared-memory tile ring (48 KB; RP_XGPU_NBUF 2..8)
constexpr int kNbufMax = 8;
constexpr int kLaneIters = 3;                     // (unused default; see xgpu_geometry)
constexpr int kMinTiles = 2;                      // smallest chunk: 2 tiles (32 KB fp32)

__device__ __forceinline__ float4 ldv(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ldg_nc(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void stv(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 div4(float4 a, float k) {
  return make_float4(__fdiv_rn(a.x, k), __fdiv_rn(a.y, k), __fdiv_rn(a.z, k), __fdiv_rn(a.w, k));
}

// ---- TMA bulk stores (cp.async.bulk global <- shared::cta) ----------------------------------
__device__ __forceinline__ void bulk_store(void* dst_global, const void* src_smem, uint32_t bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(src_smem));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_global), "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }

// flag word of (slot, src GPU, kind, chunk) in a GPU's flag array
__device__ __forceinline__ unsigned long long* flag_at(unsigned long long* base, int slot, int src, int kind,
                                                       int64_t c) {
  return base + (static_cast<int64_t>(slot) * kFlagSrc + src) * kFlagStride +
         (kind == kFlagA ? c : (kind == kFlagB ? kMaxChunks + c : 2 * kMaxChunks));
}

// Spin until *f == tag. false: the watchdog limit passed (recorded in T.err, host-mapped).
__device__ __noinline__ bool wait_flag_slow(const XTask& T, const unsigned long long* f, unsigned long long tag,
                                            int slot, int src, int kind, int64_t c) {
  const unsigned long long t0 = gtimer();
  for (unsigned n = 1;; ++n) {
    __nanosleep(32);
    if (ld_acquire_sys(f) == tag) return true;
    if (T.watchdog_ns && (n & 1023u) == 0) {
      if (T.err && *reinterpret_cast<volatile unsigned long long*>(&T.err->code)) return false;  // job failed
      if (gtimer() - t0 <= T.watchdog_ns) continue;
      if (T.err && atomicCAS(&T.err->code, 0ull, 1ull) == 0ull) {
        T.err->gpu = T.my_gpu;
        T.err->src = src;
        T.err->kind = kind;
        T.err->slot = slot;
        T.err->chunk = c;
        T.err->tag = tag;
        T.err->seen = ld_acquire_sys(f);
        __threadfence_system();
      }
      return false;
    }
  }
}
__device__ __forceinline__ bool wait_flag(const XTask& T, const unsigned long long* f, unsigned long long tag,
                                          int slot, int src, int kind, int64_t c) {
  if (ld_acquire_sys(f) == tag) return true;
  const unsigned long long t0 = T.cta_stat ? gtimer() : 0;
  const bool ok = wait_flag_slow(T, f, tag, slot, src, kind, c);
  if (T.cta_stat) atomicAdd(T.cta_stat + 4 * blockIdx.x + 2, gtimer() - t0);
  return ok;
}

// ---- element access: fp32 replicas, or bf16 replicas with fp32 arithmetic (reading R26) ----
// A "vector" is 4 consecutive elements: 16 bytes of fp32 or 8 bytes of bf16. Staged partials are
// always fp32 (the fold runs in fp32); the mean is rounded once to bf16 when stored.
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t bf_rn(float v) {  // IEEE round-to-nearest-even; NaN stays NaN
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v)));  // cvt.rn.bf16.f32, as preduce_tma.cu
}
__device__ __forceinline__ uint2 pack_bf4(float4 v) {
  return make_uint2(bf_rn(v.x) | (bf_rn(v.y) << 16), bf_rn(v.z) | (bf_rn(v.w) << 16));
}
template <bool BF>
__device__ __forceinline__ float4 ldx4(const float* base, int64_t i) {
  if constexpr (BF) {
    uint32_t a, b;
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(a), "=r"(b)
                 : "l"(reinterpret_cast<const uint16_t*>(base) + 4 * i));
    return make_float4(bf_lo(a), bf_hi(a), bf_lo(b), bf_hi(b));
  } else {
    return ldv(base + 4 * i);
  }
}
template <bool BF>
__device__ __forceinline__ float4 ldg4(const float* base, int64_t i) {
  if constexpr (BF) {
    uint32_t a, b;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(a), "=r"(b)
                 : "l"(reinterpret_cast<const uint16_t*>(base) + 4 * i));
    return make_float4(bf_lo(a), bf_hi(a), bf_lo(b), bf_hi(b));
  } else {
    return ldg_nc(base + 4 * i);
  }
}
template <bool BF>
__device__ __forceinline__ void stx4(float* base, int64_t i, float4 v) {
  if constexpr (BF) {
    const uint2 w = pack_bf4(v);
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(reinterpret_cast<uint16_t*>(base) + 4 * i), "r"(w.x),
                 "r"(w.y)
                 : "memory");
  } else {
    stv(base + 4 * i, v);
  }
}
template <bool BF>
__device__ __forceinline__ float ldx1(const float* base, int64_t j) {
  if constexpr (BF) return __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(base)[j]) << 16);
  else return base[j];
}
template <bool BF>
__device__ __forceinline__ void stx1(float* base, int64_t j, float v) {
  if constexpr (BF) reinterpret_cast<uint16_t*>(base)[j] = static_cast<uint16_t>(bf_rn(v));
  else base[j] = v;
}
template <bool MOM, bool BF>
__device__ __forceinline__ float step1x(const float* x, const MemberUpdate& u, int64_t j) {
  if constexpr (BF) {
    const float xv = ldx1<true>(x, j);
    return u.g == nullptr ? xv : step_sgd(xv, ldx1<true>(u.g, j), u.lr);
  } else {
    return step1<MOM>(x[j], u, j);
  }
}

// Local partials of my p.m (<= M) members for U rows of one tile: vector i = i0 + u * kRowF4,
// left fold in ascending worker id, alg1 step 2 applied (momentum buffers updated: each
// element's partial is computed exactly once, in its A or B stage). The loads of MB members
// of the U rows are issued before they are folded (MB = 2 beyond two members: registers).
template <int M, int U, bool MOM, bool BF>
__device__ __forceinline__ void partials(const XPart& p, int64_t i0, int64_t hi, float4 (&s)[U]) {
  constexpr int MB = M <= 2 ? M : 2;
#pragma unroll
  for (int m0 = 0; m0 < M; m0 += MB) {
    if (m0 >= p.m) break;
    float4 xv[U][MB], gv[U][MB], vv[U][MOM ? MB : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * kRowF4;
      if (i < hi) {
#pragma unroll
        for (int b = 0; b < MB; ++b) {
          const int m = m0 + b;
          if (m < p.m) {
            xv[u][b] = ldx4<BF>(p.x[m], i);
            if (p.u[m].g) gv[u][b] = ldg4<BF>(p.u[m].g, i);
            if constexpr (MOM)
              if (p.u[m].v) vv[u][b] = ldv(p.u[m].v + 4 * i);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * kRowF4;
      if (i < hi) {
#pragma unroll
        for (int b = 0; b < MB; ++b) {
          const int m = m0 + b;
          if (m < p.m) {
            float4 vm = vv[u][MOM ? b : 0];
            const float4 y = step4<MOM>(xv[u][b], gv[u][b], vm, p.u[m]);
            if constexpr (MOM)
              if (p.u[m].v && p.u[m].g) stv(p.u[m].v + 4 * i, vm);
            s[u] = m == 0 ? y : add4(s[u], y);
          }
        }
      }
    }
  }
}
template <int M, bool MOM, bool BF>
__device__ __forceinline__ float partial1(const XPart& p, int64_t j) {
  float s = step1x<MOM, BF>(p.x[0], p.u[0], j);
#pragma unroll
  for (int m = 1; m < M; ++m)
    if (m < p.m) s = __fadd_rn(s, step1x<MOM, BF>(p.x[m], p.u[m], j));
  return s;
}

// Chunk c of slice o: vector range [lo, hi); the last chunk of the last slice also carries the
// n mod 4 scalar tail.
struct ChunkRange {
  int64_t lo, hi;
  bool tail;
};
__device__ __forceinline__ int64_t slice_lo(const XPart& p, int o) { return min(static_cast<int64_t>(o) * p.S4, p.n4); }
__device__ __forceinline__ ChunkRange chunk_range(const XPart& p, int o, int64_t c) {
  const int64_t slo = slice_lo(p, o), shi = min(static_cast<int64_t>(o + 1) * p.S4, p.n4);
  ChunkRange r;
  // balanced big chunks: tiles [c CH / nbig, (c+1) CH / nbig); then nsmall chunks of tail_w tiles
  const int64_t nbig = p.nch - p.nsmall;
  const int64_t t_lo = c < nbig ? (c * p.CH) / nbig : p.CH + (c - nbig) * p.tail_w;
  const int64_t t_hi = c < nbig ? ((c + 1) * p.CH) / nbig : t_lo + p.tail_w;
  r.lo = min(slo + t_lo * 1024, shi);
  r.hi = min(slo + t_hi * 1024, shi);
  r.tail = (o == p.kp - 1) && (c == p.nch - 1) && p.rem > 0;
  return r;
}
// float offset of (row d, vector i relative to the slice start) in a staging region: row d
// holds the partials GPU d sends for the owner's slice; S4 + 1 vectors per row so the tail
// scalars fit after the slice's vector range.
__device__ __forceinline__ int64_t stage_off(const XPart& p, int d, int64_t i_rel) {
  return (static_cast<int64_t>(d) * (p.S4 + 1) + i_rel) * 4;
}

// Shared-memory tile ring of nbuf tiles: `slot` counts tiles issued by this CTA; a tile buffer is
// reused only after the bulk store that read it nbuf tiles ago has finished reading (thread 0
// waits, the barrier publishes). Every tile commits exactly one bulk group.
__device__ __forceinline__ void bulk_wait_read_n(int n) {
  switch (n) {
    case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group.read 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.bulk.wait_group.read 6;" ::: "memory"); break;
    case 7: asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
  }
}
__device__ __forceinline__ void stat_add(unsigned long long* st, int k, unsigned long long t0) {
  if (st) atomicAdd(st + 4 * blockIdx.x + k, gtimer() - t0);
}
__device__ __forceinline__ float4* acquire_tile(float4* smem, int& slot, int nbuf, unsigned long long* st) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = st ? gtimer() : 0;
    bulk_wait_read_n(nbuf - 1);
    stat_add(st, 0, t0);
  }
  __syncthreads();
  float4* b = smem + (slot % nbuf) * kTileF4;
  ++slot;
  return b;
}

// A(o, c): my partial of chunk c of slice o -> owner o's staging row me (NVLink).
template <int M, int U, bool MOM, bool BF>
__device__ void stage_A(const XPart& p, int o, int64_t c, float4* smem, int& slot, int& ncommit, int nbuf,
                        unsigned long long* st) {
  const ChunkRange r = chunk_range(p, o, c);
  const int64_t slo = slice_lo(p, o);
  float* dst = p.stage[o];
  for (int64_t t0 = r.lo; t0 < r.hi; t0 += kTileF4) {
    float4* sb = acquire_tile(smem, slot, nbuf, st);
#pragma unroll
    for (int r0 = 0; r0 < kTileRows; r0 += U) {
      float4 s[U];
      const int64_t i0 = t0 + r0 * kRowF4 + threadIdx.x;
      partials<M, U, MOM, BF>(p, i0, r.hi, s);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * kRowF4 < r.hi) sb[(r0 + u) * kRowF4 + threadIdx.x] = s[u];
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t cnt = min(kTileF4, r.hi - t0);
      bulk_store(dst + stage_off(p, p.me, t0 - slo), sb, static_cast<uint32_t>(cnt * 16));  // NVLink
      bulk_commit();
      ++ncommit;
    }
  }
  if (r.tail && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    dst[stage_off(p, p.me, p.n4 - slo) + threadIdx.x] = partial1<M, MOM, BF>(p, j);  // NVLink (plain store)
  }
}

// B(c): fold my slice's chunk c over all GPUs, divide, store locally and push to every peer.
template <int M, int U, bool MOM, bool BF, int KPM>
__device__ void stage_B(const XPart& p, int64_t c, float4* smem, int& slot, int& ncommit, int nbuf,
                        unsigned long long* st) {
  const int o = p.me;
  const ChunkRange r = chunk_range(p, o, c);
  const int64_t slo = slice_lo(p, o);
  const float* stage = p.stage[o];  // my staging region (local)
  const float kf = static_cast<float>(p.k_total);
  for (int64_t t0 = r.lo; t0 < r.hi; t0 += kTileF4) {
    float4* sb = acquire_tile(smem, slot, nbuf, st);
#pragma unroll
    for (int r0 = 0; r0 < kTileRows; r0 += U) {
      const int64_t i0 = t0 + r0 * kRowF4 + threadIdx.x;
      float4 mine[U];
      float4 part[U][KPM];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * kRowF4;
        if (i < r.hi)
#pragma unroll
          for (int d = 0; d < KPM; ++d)
            if (d < p.kp && d != o) part[u][d] = ldv(stage + stage_off(p, d, i - slo));
      }
      partials<M, U, MOM, BF>(p, i0, r.hi, mine);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * kRowF4;
        if (i < r.hi) {
          float4 s = o == 0 ? mine[u] : part[u][0];
#pragma unroll
          for (int d = 1; d < KPM; ++d)
            if (d < p.kp) s = add4(s, d == o ? mine[u] : part[u][d]);
          const float4 xbar = div4(s, kf);
#pragma unroll
          for (int m = 0; m < M; ++m)
            if (m < p.m) stx4<BF>(p.x[m], i, xbar);
          if constexpr (BF) {
            reinterpret_cast<uint2*>(sb)[(r0 + u) * kRowF4 + threadIdx.x] = pack_bf4(xbar);
            // bulk copies move multiples of 16 bytes: an odd last bf16 vector goes by plain store
            if (((r.hi - t0) & 1) && i == r.hi - 1 && r.hi - t0 <= kTileF4)
              for (int d = 0; d < p.kp; ++d)
                if (d != o) stx4<true>(p.xfirst[d], i, xbar);  // NVLink
          } else {
            sb[(r0 + u) * kRowF4 + threadIdx.x] = xbar;
          }
        }
      }
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t cnt = min(kTileF4, r.hi - t0);
      const uint32_t bytes = static_cast<uint32_t>(BF ? (cnt & ~1LL) * 8 : cnt * 16);
      for (int j = 1; j < p.kp; ++j) {
        const int d = (o + j) % p.kp;  // spread the pushes over the peers
        void* dst = BF ? static_cast<void*>(reinterpret_cast<uint16_t*>(p.xfirst[d]) + 4 * t0)
                       : static_cast<void*>(p.xfirst[d] + 4 * t0);
        if (bytes) bulk_store(dst, sb, bytes);  // NVLink
      }
      bulk_commit();
      ++ncommit;
    }
  }
  if (r.tail && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    const int64_t so = p.n4 - slo;
    const float mine = partial1<M, MOM, BF>(p, j);
    float s = o == 0 ? mine : stage[stage_off(p, 0, so) + threadIdx.x];
    for (int d = 1; d < p.kp; ++d) s = __fadd_rn(s, d == o ? mine : stage[stage_off(p, d, so) + threadIdx.x]);
    const float xbar = __fdiv_rn(s, kf);
    for (int m = 0; m < p.m; ++m) stx1<BF>(p.x[m], j, xbar);
    for (int d = 0; d < p.kp; ++d)
      if (d != o) stx1<BF>(p.xfirst[d], j, xbar);
  }
}

// C(o, c): xbar of chunk c of slice o has landed in my first local member: copy it to the others.
template <int M, bool BF>
__device__ void stage_C(const XPart& p, int o, int64_t c) {
  const ChunkRange r = chunk_range(p, o, c);
  constexpr int U = 4;
  for (int64_t t0 = r.lo; t0 < r.hi; t0 += kRowF4 * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kRowF4 + threadIdx.x;
      if (i < r.hi) v[u] = ldx4<BF>(p.x[0], i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kRowF4 + threadIdx.x;
      if (i < r.hi)
#pragma unroll
        for (int m = 1; m < M; ++m)
          if (m < p.m) stx4<BF>(p.x[m], i, v[u]);  // exact for bf16 (already rounded)
    }
  }
  if (r.tail && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    const float v = ldx1<BF>(p.x[0], j);
    for (int m = 1; m < p.m; ++m) stx1<BF>(p.x[m], j, v);
  }
}

__device__ __forceinline__ void prof_rec(const XTask& T, int pi, int kind, int64_t c, unsigned long long ts,
                                         unsigned long long tr) {
  if (T.prof && threadIdx.x == 0) {
    XItemRecord rec;
    rec.t_start = ts;
    rec.t_ready = tr;
    rec.t_end = gtimer();
    rec.meta = (static_cast<unsigned long long>(kind) << 62) | (static_cast<unsigned long long>(pi) << 56) |
               (static_cast<unsigned long long>(blockIdx.x & 0xFFFFFF) << 32) | static_cast<unsigned long long>(c);
    T.prof[(static_cast<int64_t>(pi) * 3 + kind) * kMaxChunks + c] = rec;
  }
}

// cp.async.bulk.wait_group takes an immediate: wait until at most n (clamped to 63) of this
// thread's most recent bulk groups are pending.
__device__ __forceinline__ void bulk_wait_pending(int n) {
  switch (n < 63 ? n : 63) {
#define RP_W(k) \
  case k: asm volatile("cp.async.bulk.wait_group " #k ";" ::: "memory"); break;
#define RP_W8(k) RP_W(k) RP_W(k + 1) RP_W(k + 2) RP_W(k + 3) RP_W(k + 4) RP_W(k + 5) RP_W(k + 6) RP_W(k + 7)
    RP_W8(0) RP_W8(8) RP_W8(16) RP_W8(24) RP_W8(32) RP_W8(40) RP_W8(48) RP_W8(56)
#undef RP_W8
#undef RP_W
  }
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Publish the flags of the stores issued in an earlier iteration (thread 0): those bulk groups
// have completed (caller waited), fence.proxy.async makes the async-proxy writes visible to the
// generic proxy, one fence.acq_rel.sys + relaxed stores form the release (cumulative: the other
// threads' plain tail stores are ordered by the barrier before it).
__device__ __forceinline__ void post_flags(const XTask& T, const XPart& p, int64_t cA, int64_t cB) {
  if (cA < 0 && cB < 0) return;
  fence_async_all();
  fence_acq_rel_sys();
  if (cA >= 0)
    for (int j = 1; j < p.kp; ++j) {
      const int o = (p.me + j) % p.kp;
      st_relaxed_sys(flag_at(p.pflags[o], p.slot, T.my_gpu, kFlagA, cA), p.tag[o]);
    }
  if (cB >= 0)
    for (int d = 0; d < p.kp; ++d)
      if (d != p.me) st_relaxed_sys(flag_at(p.pflags[d], p.slot, T.my_gpu, kFlagB, cB), p.tag[d]);
}

// One lane of part pi: the pipelined iterations. false = a flag wait hit the watchdog.
//
// Iteration i issues A(c_i), B(c_{i-2}), C(c_{i-4}) and then publishes the flags of iteration
// i-1's stores once those have completed, while iteration i's stores are still on the wire
// (deferred signalling: a CTA never drains its NVLink pushes to post a flag; waiting for all of
// them cost 10-25 % at 32-128 KB per flag, profiles/r02/bulk_push_probe_2gpu.txt). A(c) flags
// are posted at the end of iteration c+1, so B(c) runs in iteration c+2 (the peers' flags are
// one iteration old by then); B(c) flags at the end of c+3, so C(c) runs in c+4.
template <int M, int UA, int UB, bool MOM, bool BF, int KPM>
__device__ bool run_lane(const XTask& T, int pi, int lane, float4* smem, int& slot, unsigned long long& ready_seen,
                         int* s_abort) {
  const XPart& p = T.part[pi];
  const int64_t iters = lane < p.nch ? (p.nch - 1 - lane) / kXLanes + 1 : 0;
  int64_t pA = -1, pB = -1;  // chunks whose stores the previous iteration issued (flags pending)
  for (int64_t i = 0; i < (iters ? iters + 4 : 0); ++i) {
    const int64_t cA = i < iters ? lane + i * kXLanes : -1;
    const int64_t cB = (i >= 2 && i - 2 < iters) ? lane + (i - 2) * kXLanes : -1;
    const int64_t cC = (i >= 4 && i - 4 < iters) ? lane + (i - 4) * kXLanes : -1;
    int ncommit = 0;  // bulk groups committed in this iteration (thread 0)
    unsigned long long ts = 0;
    if (cA >= 0) {
      if (T.prof && threadIdx.x == 0) ts = gtimer();
      for (int j = 1; j < p.kp; ++j) {
        const int o = (p.me + j) % p.kp;  // spread the pushes over the owners
        const unsigned long long bit = 1ull << (8 * pi + o);
        if (threadIdx.x == 0 && !(ready_seen & bit)) {
          if (!wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[o], kFlagReady, 0), p.tag[o], p.slot, p.gpu[o],
                         kFlagReady, 0))
            *s_abort = 1;
          ready_seen |= bit;
        }
        __syncthreads();
        if (*s_abort) return false;
        stage_A<M, UA, MOM, BF>(p, o, cA, smem, slot, ncommit, T.nbuf, T.cta_stat);
      }
      prof_rec(T, pi, 0, cA, ts, ts);
    }
    if (cB >= 0) {
      unsigned long long tr = 0;
      if (T.prof && threadIdx.x == 0) ts = gtimer();
      if (threadIdx.x == 0)
        for (int d = 0; d < p.kp; ++d)
          if (d != p.me && !wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[d], kFlagA, cB), p.tag[d], p.slot,
                                      p.gpu[d], kFlagA, cB)) {
            *s_abort = 1;
            break;
          }
      __syncthreads();
      if (*s_abort) return false;
      if (T.prof && threadIdx.x == 0) tr = gtimer();
      stage_B<M, UB, MOM, BF, KPM>(p, cB, smem, slot, ncommit, T.nbuf, T.cta_stat);
      prof_rec(T, pi, 1, cB, ts, tr);
    }
    if (cC >= 0) {
      for (int j = 1; j < p.kp; ++j) {
        const int o = (p.me + j) % p.kp;
        unsigned long long tr = 0;
        if (T.prof && threadIdx.x == 0) ts = gtimer();
        if (threadIdx.x == 0 && !wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[o], kFlagB, cC), p.tag[o], p.slot,
                                           p.gpu[o], kFlagB, cC))
          *s_abort = 1;
        __syncthreads();
        if (*s_abort) return false;
        if (T.prof && threadIdx.x == 0) tr = gtimer();
        if (p.m > 1) stage_C<M, BF>(p, o, cC);
        if (j == p.kp - 1) prof_rec(T, pi, 2, cC, ts, tr);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long t0 = T.cta_stat ? gtimer() : 0;
      bulk_wait_pending(ncommit);  // the previous iteration's groups have completed
      stat_add(T.cta_stat, 1, t0);
      post_flags(T, p, pA, pB);
    }
    pA = cA;
    pB = cB;
  }
  if (threadIdx.x == 0 && (pA >= 0 || pB >= 0)) {  // (never: the last iterations issue only C)
    bulk_wait_all();
    post_flags(T, p, pA, pB);
  }
  return true;
}

// The kernel body for one GPU's task, run by CTAs cta = 0 .. ncta-1.
template <int M, int UA, int UB, bool MOM, bool BF, int KPM>
__device__ __forceinline__ void xgpu_body(const XTask& T, int cta, int ncta) {
  static_assert(!BF || !MOM, "bf16 replicas: plain SGD only");
  extern __shared__ float4 xsmem[];
  __shared__ int s_abort;
  if (threadIdx.x == 0) s_abort = 0;
  if (cta == 0 && threadIdx.x == 0) {
    // READY: my staging is free for these groups (my previous kernel has finished)
    for (int pi = 0; pi < T.nparts; ++pi) {
      const XPart& p = T.part[pi];
      for (int d = 0; d < p.kp; ++d)
        if (d != p.me) st_release_sys(flag_at(p.pflags[d], p.slot, T.my_gpu, kFlagReady, 0), p.tag[d]);
    }
  }
  __syncthreads();
  const unsigned long long t_begin = T.cta_stat ? gtimer() : 0;
  int slot = 0;
  unsigned long long ready_seen = 0;  // bit 8*pi + o: READY of part pi's owner o observed (thread 0)
  const int total = T.nparts * kXLanes;
  bool ok = true;
  for (int idx = cta; ok && idx < total; idx += ncta)
    ok = run_lane<M, UA, UB, MOM, BF, KPM>(T, idx % T.nparts, idx / T.nparts, xsmem, slot, ready_seen, &s_abort);
  if (threadIdx.x == 0) {
    bulk_wait_all();  // never leave with a bulk store reading shared memory
    stat_add(T.cta_stat, 3, t_begin);
  }
}

template <int M, int UA, int UB, bool MOM, bool BF, int KPM>
__global__ void __launch_bounds__(kXThreads, (M >= 4 || MOM) ? 1 : RP_XGPU_MINB)
    xgpu_kernel(const __grid_constant__ XTask T) {
  xgpu_body<M, UA, UB, MOM, BF, KPM>(T, blockIdx.x, gridDim.x);
}

// Emulation (RP_FLAG_EMULATE): every virtual GPU's task in ONE cooperative launch on one device,
// virtual GPU v on CTAs v, v + V, v + 2V, ... (all co-resident: a spinning CTA never starves the
// CTA it waits for; separate spinning launches on one GPU are not guaranteed to run together).
template <int M, int UA, int UB, bool MOM, bool BF, int KPM>
__global__ void __launch_bounds__(kXThreads, (M >= 4 || MOM) ? 1 : RP_XGPU_MINB)
    xgpu_emul_kernel(const XTask* __restrict__ tasks, int V) {
  const int v = blockIdx.x % V;
  xgpu_body<M, UA, UB, MOM, BF, KPM>(tasks[v], blockIdx.x / V, gridDim.x / V);
}

int g_sms = 0;
int env_int(const char* name, int def) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : def;
}

constexpr size_t kSmemMax = static_cast<size_t>(kNbufMax) * kTileF4 * sizeof(float4);
int nbuf_setting() {
  static const int v = std::min(kNbufMax, std::max(2, env_int("RP_XGPU_NBUF", kNbufDefault)));
  return v;
}
size_t smem_bytes(int nbuf) { return static_cast<size_t>(nbuf) * kTileF4 * sizeof(float4); }


int sm_count() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

// 48 KB of dynamic shared memory + the static words exceed the default 48 KB per-CTA limit
template <typename F>
bool smem_attr(F fn) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemMax)) ==
         cudaSuccess;
}

template <int M, int UA, int UB, bool MOM, bool BF, int KPM>
int launch_m(XTask& T, cudaStream_t stream, std::string* err) {
  static int occ = 0;
  if (occ == 0) {
    if (!smem_attr(xgpu_kernel<M, UA, UB, MOM, BF, KPM>)) {
      *err = "xgpu: shared memory attribute";
      return RP_ECUDA;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, xgpu_kernel<M, UA, UB, MOM, BF, KPM>, kXThreads,
                                                      smem_bytes(nbuf_setting())) !=
            cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  int64_t grid = static_cast<int64_t>(sm_count()) * occ;  // every CTA co-resident
  static int cps = -1;
  if (cps < 0) cps = env_int("RP_XGPU_CTAS_PER_SM", 0);
  if (cps > 0) grid = std::min<int64_t>(grid, static_cast<int64_t>(sm_count()) * cps);
  if (T.max_ctas > 0) grid = std::min<int64_t>(grid, T.max_ctas);
  grid = std::max<int64_t>(1, std::min<int64_t>(grid, static_cast<int64_t>(T.nparts) * kXLanes));
  T.nbuf = nbuf_setting();
  xgpu_kernel<M, UA, UB, MOM, BF, KPM><<<static_cast<int>(grid), kXThreads, smem_bytes(T.nbuf), stream>>>(T);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("xgpu kernel launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

template <int M, int UA, int UB, bool MOM, bool BF, int KPM>
int launch_emul_m(const XTask* d_tasks, int V, int max_parts, cudaStream_t stream, std::string* err) {
  auto fn = xgpu_emul_kernel<M, UA, UB, MOM, BF, KPM>;
  static bool attr = false;
  if (!attr) {
    if (!smem_attr(fn)) {
      *err = "xgpu emulation: shared memory attribute";
      return RP_ECUDA;
    }
    attr = true;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kXThreads, smem_bytes(nbuf_setting())) != cudaSuccess ||
      occ < 1) {
    *err = "xgpu emulation: occupancy query failed";
    return RP_ECUDA;
  }
  const int64_t resident = static_cast<int64_t>(sm_count()) * occ;
  const int64_t per = std::min<int64_t>(resident / V, static_cast<int64_t>(max_parts) * kXLanes);
  if (per < 1) {
    *err = "xgpu emulation: more virtual GPUs than resident CTAs";
    return RP_EINVAL;
  }
  int grid = static_cast<int>(per * V);
  void* args[] = {const_cast<XTask**>(&d_tasks), &V};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(kXThreads),
                                                    args, smem_bytes(nbuf_setting()), stream);
  if (e != cudaSuccess) {
    *err = std::string("xgpu emulation cooperative launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

// Instantiation choice: M bounds the local member count of every part, KPM the GPU count of
// every group; UA / UB = rows per register batch in the A / B stages (<= 8 16-byte loads in
// flight per thread per batch, no spills at 128 registers).
template <bool EMU>
int dispatch(XTask& T, const XTask* d_tasks, int V, int max_parts, cudaStream_t s, std::string* err, int mmax,
             int kpmax, bool mom) {
#define RP_XL(M, UA, UB, MOM, BF, KPM)                                                 \
  return EMU ? launch_emul_m<M, UA, UB, MOM, BF, KPM>(d_tasks, V, max_parts, s, err) \
             : launch_m<M, UA, UB, MOM, BF, KPM>(T, s, err)
  if (T.bf16) {
    if (kpmax <= 2 && !EMU) {
      if (mmax <= 1) RP_XL(1, 4, 2, false, true, 2);
      if (mmax <= 2) RP_XL(2, 2, 1, false, true, 2);
      if (mmax <= 4) RP_XL(4, 1, 1, false, true, 2);
      RP_XL(8, 1, 1, false, true, 2);
    }
    if (mmax <= 1) RP_XL(1, 4, 1, false, true, 8);
    if (mmax <= 2) RP_XL(2, 2, 1, false, true, 8);
    if (mmax <= 4) RP_XL(4, 1, 1, false, true, 8);
    RP_XL(8, 1, 1, false, true, 8);
  }
  if (mom) {
    if (mmax <= 1) RP_XL(1, 2, 1, true, false, 8);
    if (mmax <= 2) RP_XL(2, 1, 1, true, false, 8);
    if (mmax <= 4) RP_XL(4, 1, 1, true, false, 8);
    RP_XL(8, 1, 1, true, false, 8);
  }
  if (kpmax <= 2 && !EMU) {
    if (mmax <= 1) RP_XL(1, 4, 2, false, false, 2);
    if (mmax <= 2) RP_XL(2, 2, 1, false, false, 2);
    if (mmax <= 4) RP_XL(4, 1, 1, false, false, 2);
    RP_XL(8, 1, 1, false, false, 2);
  }
  if (kpmax <= 4 && !EMU) {
    if (mmax <= 1) RP_XL(1, 4, 1, false, false, 4);
    if (mmax <= 2) RP_XL(2, 2, 1, false, false, 4);
    if (mmax <= 4) RP_XL(4, 1, 1, false, false, 4);
    RP_XL(8, 1, 1, false, false, 4);
  }
  if (mmax <= 1) RP_XL(1, 4, 1, false, false, 8);
  if (mmax <= 2) RP_XL(2, 2, 1, false, false, 8);
  if (mmax <= 4) RP_XL(4, 1, 1, false, false, 8);
  RP_XL(8, 1, 1, false, false, 8);
#undef RP_XL
}

template <int M, int UA, int UB, bool MOM, bool BF, int KPM>
void x_touch() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, xgpu_kernel<M, UA, UB, MOM, BF, KPM>);
  cudaFuncGetAttributes(&a, xgpu_emul_kernel<M, UA, UB, MOM, BF, KPM>);
}

int check_task(const XTask& T, int* mmax, int* kpmax, bool* mom, std::string* err) {
  if (T.nparts < 1 || T.nparts > kMaxXParts) {
    *err = "xgpu: bad part count";
    return RP_EINVAL;
  }
  for (int pi = 0; pi < T.nparts; ++pi) {
    const XPart& p = T.part[pi];
    if (p.m < 1 || p.m > kMaxXLocal || p.kp < 2 || p.kp > kMaxXGpus || p.me < 0 || p.me >= p.kp || p.nch < 1 ||
        p.nch > kMaxChunks) {
      *err = "xgpu: bad part descriptor";
      return RP_EINVAL;
    }
    for (int d = 0; d < p.kp; ++d)
      if (!p.stage[d] || !p.xfirst[d] || !p.pflags[d] || (reinterpret_cast<uintptr_t>(p.xfirst[d]) & 15) ||
          (reinterpret_cast<uintptr_t>(p.stage[d]) & 15) || (d != p.me && p.tag[d] == 0)) {
        *err = "xgpu: peer pointers missing (call rp_peer_import), misaligned, or zero tag";
        return RP_EINVAL;
      }
    *mmax = std::max(*mmax, p.m);
    *kpmax = std::max(*kpmax, p.kp);
    for (int m = 0; m < p.m; ++m) *mom = *mom || (p.u[m].v && p.u[m].g);
  }
  if (T.bf16 && *mom) {
    *err = "xgpu: bf16 replicas take plain SGD";
    return RP_EINVAL;
  }
  if (T.nlocal < 0 || T.nlocal > kMaxXLocalGroups) {
    *err = "xgpu: bad fused-group count";
    return RP_EINVAL;
  }
  for (int gi = 0; gi < T.nlocal; ++gi) {
    const XLocalGroup& G = T.lg[gi];
    if (G.k < 1 || G.k > kMaxFusedK) {
      *err = "xgpu: fused intra-GPU groups have 1..4 members";
      return RP_EINVAL;
    }
    for (int m = 0; m < G.k; ++m) {
      if (!G.x[m] || (reinterpret_cast<uintptr_t>(G.x[m]) & 15) || (reinterpret_cast<uintptr_t>(G.u[m].g) & 15)) {
        *err = "xgpu: fused group replica / gradient pointers must be non-null and 16-byte aligned";
        return RP_EINVAL;
      }
      *mom = *mom || (G.u[m].v && G.u[m].g);
    }
    *mmax = std::max(*mmax, static_cast<int>(G.k));  // L jobs need 2k operand slots (2M >= 2k)
  }
  if (T.nlocal > 0 && (*mom || use_v2())) {
    *err = "xgpu: fused intra-GPU groups need the warp-specialized kernel (plain SGD, RP_XGPU_V2 unset)";
    return RP_EINVAL;
  }
  return RP_OK;
}

}  // namespace

// RP_XGPU_V2=1: the register (LDG/STG) version of this file for plain SGD too (comparison);
// momentum steps always take it (their buffers are read and written per member)
int sig2_setting() {  // RP_XGPU_SIG2: two SIG jobs per lane iteration in the warp-specialized kernel
  static const int v = env_int("RP_XGPU_SIG2", 1) != 0;
  return v;
}
int blag_setting() {  // RP_XGPU_BLAG: iterations between a chunk's A and B stages (tuning)
  // one SIG per iteration: >= 2, 3 best (profiles/r02/sweep_blag_2gpu.txt); two SIGs: >= 1, 1 best
  // (2 with early A flags measured one 1.5 ms/step cfg3 run at N = 4, profiles/r02/sweep_iters_early_a_4gpu.txt)
  static const int v = std::max(sig2_setting() ? 1 : 2, std::min(6, env_int("RP_XGPU_BLAG", sig2_setting() ? 1 : 3)));
  return v;
}

// RP_XGPU_LOOKAHEAD = 1 (experiment, off): under dynamic claiming, when a B block's A flags are not
// all posted, the producer claims and pushes the next chunk's A block first. Parity holds (emulated
// and 2/4-GPU suites) but it is slower everywhere (ResNet-50 xall at N = 2: 0.61 vs 0.68 of 770 GB/s;
// configs[3] layout at N = 4: 5,140 vs 5,435 worker-steps/s): the B block a peer waits for is pushed
// later, profiles/r02/sweep_lookahead_{2,4}gpu.txt. So 0.
// RP_XGPU_EARLY_A (default 1): under dynamic claiming a chunk's A flags are posted from a SIG after the
// first tile of the iteration's B block instead of at the iteration's end, so the peers' B blocks of
// that chunk wait less (per-iteration timelines: B blocks waited for A flags posted behind a whole B
// block, profiles/r02/timeline_sig_*.txt). Measured (profiles/r02/sweep_early_a_{2,4}gpu.txt, two runs
// each): N = 4 configs[3] layout 5,439 / 5,374 -> 5,587 / 5,581, xall +5-9 %, cfg3 +1 %, r50x8 -0.5 %
// (noise); N = 2 xall / cfg3 +3 %, r50x8 and configs[3] layout unchanged.
int early_a_setting() {
  static const int v = env_int("RP_XGPU_EARLY_A", 1) != 0;
  return v;
}

int lookahead_setting() {
  static const int v = env_int("RP_XGPU_LOOKAHEAD", 0) != 0;
  return v;
}

bool use_v2() {
  static const int v = env_int("RP_XGPU_V2", 0);
  return v == 1;
}

void xgpu_geometry(XPart& p, int64_t n) {
  p.n4 = n / 4;
  p.rem = static_cast<int32_t>(n - 4 * p.n4);
  p.S4 = ((p.n4 + p.kp - 1) / p.kp + kTileF4 - 1) / kTileF4 * kTileF4;
  p.S4 = std::max<int64_t>(p.S4, kTileF4);
  // every lane gets the same number of chunks (kLaneIters of them) and chunk sizes differ by at
  // most one tile (a fixed chunk size left up to 28 % more work on some lanes than the average,
  // and the slowest lane sets the kernel time); chunks of >= kMinTiles tiles on average, at most
  // kMaxChunks. RP_XGPU_ITERS / RP_XGPU_MIN_TILES override (tuning; every rank of a job must see
  // the same values: the geometry must agree across GPUs)
  // Default: about 4 tiles (64 KB) per chunk, 2..6 chunks per lane -- ResNet-50 slices take 2-3
  // chunks per lane, VGG-16 slices 6 (6 gave +7 % at VGG size: profiles/r02/sweep_dyn_2gpu.txt).
  // The floor was 3 while A flags were posted at the iteration's end (2 lost 12 % on the 8-worker
  // problem at N = 4, r02/final_4gpu/); with early A flags 2 is as good or better at ResNet-50 size
  // (N = 4, medians of three alternated runs: r50x8 18,055 vs 17,300, cfg3 14,611 vs 14,519;
  // profiles/r02/sweep_iters_early_a_4gpu*.txt).
  static const int iters_env = env_int("RP_XGPU_ITERS", 0);
  static const int min_tiles = std::max(1, env_int("RP_XGPU_MIN_TILES", kMinTiles));
  const int64_t tiles = p.S4 / kTileF4;
  const int iters = iters_env > 0 ? iters_env
                                  : static_cast<int>(std::max<int64_t>(
                                        2, std::min<int64_t>(6, (tiles + kXLanes * 3) / (kXLanes * 4))));
  // RP_XGPU_TAIL = t > 0 (experiment, off): the last t chunks are RP_XGPU_TAIL_TILES tiles each
  // (default 1), taken last under dynamic claiming to shorten the kernel's tail; RP_XGPU_TAIL_KEEP=1
  // takes them out of the big chunks' count (same number of chunks, so the same flag overhead).
  // t = 296 single tiles on top of the big chunks measured slower (ResNet-50 xall 0.62 vs 0.67 of
  // 770 GB/s: the per-chunk flag and SIG overhead outweighs the shorter tail,
  // profiles/r02/sweep_tail_2gpu.txt); carved out of the big chunks (KEEP=1) at N = 4: 296 x 2 tiles
  // cfg3 +4 %, xall +3 %, r50x8 -1 %, configs[3] layout -2 %; 296 x 1 and 592 x 1 slower
  // (profiles/r02/sweep_tail_keep_4gpu.txt, one run each, within the box spread), so 0.
  static const int tail_env = env_int("RP_XGPU_TAIL", 0);
  static const int tail_w = std::max(1, env_int("RP_XGPU_TAIL_TILES", 1));
  static const int tail_keep = env_int("RP_XGPU_TAIL_KEEP", 0);
  const int64_t nsmall = std::min<int64_t>(std::max(0, tail_env), tiles / (4 * tail_w));
  const int64_t tb = tiles - nsmall * tail_w;
  int64_t nch = static_cast<int64_t>(kXLanes) * iters;
  nch = std::min<int64_t>(nch, std::max<int64_t>(1, tb / min_tiles));
  nch = std::min<int64_t>(nch, kMaxChunks - nsmall);
  if (nch > kXLanes) nch = nch / kXLanes * kXLanes;  // whole rounds of lanes
  if (tail_keep && nsmall > 0 && nch - nsmall >= kXLanes) nch -= nsmall;
  p.CH = tb;
  p.nsmall = static_cast<int32_t>(nsmall);
  p.tail_w = tail_w;
  p.nch = std::max<int64_t>(1, nch) + nsmall;
}

int64_t xgpu_stage_region_bytes(int64_t n) {
  // kp rows of (S4 + 1) vectors, S4 <= n4/kp + tile: at most 4n + 16 * kp * (tile + 2)
  return 4 * n + 16LL * kMaxXGpus * (kTileF4 + 2);
}

void preload_xgpu() {  // every instantiation dispatch() can pick (see preload_xgpu_ws)
#define RP_T(M, UA, UB, MOM, BF, KPM) x_touch<M, UA, UB, MOM, BF, KPM>()
  RP_T(1, 4, 2, false, true, 2); RP_T(2, 2, 1, false, true, 2); RP_T(4, 1, 1, false, true, 2);
  RP_T(8, 1, 1, false, true, 2); RP_T(1, 4, 1, false, true, 8); RP_T(2, 2, 1, false, true, 8);
  RP_T(4, 1, 1, false, true, 8); RP_T(8, 1, 1, false, true, 8); RP_T(1, 2, 1, true, false, 8);
  RP_T(2, 1, 1, true, false, 8); RP_T(4, 1, 1, true, false, 8); RP_T(8, 1, 1, true, false, 8);
  RP_T(1, 4, 2, false, false, 2); RP_T(2, 2, 1, false, false, 2); RP_T(4, 1, 1, false, false, 2);
  RP_T(8, 1, 1, false, false, 2); RP_T(1, 4, 1, false, false, 4); RP_T(2, 2, 1, false, false, 4);
  RP_T(4, 1, 1, false, false, 4); RP_T(8, 1, 1, false, false, 4); RP_T(1, 4, 1, false, false, 8);
  RP_T(2, 2, 1, false, false, 8); RP_T(4, 1, 1, false, false, 8); RP_T(8, 1, 1, false, false, 8);
#undef RP_T
}

int launch_xgpu(XTask& T, void* stream, std::string* err) {
  int mmax = 0, kpmax = 0;
  bool mom = false;
  const int rc = check_task(T, &mmax, &kpmax, &mom, err);
  if (rc != RP_OK) return rc;
  T.blag = blag_setting();
  T.sig2 = sig2_setting();
  T.lookahead = lookahead_setting();
  T.early_a = early_a_setting();
  if (!mom && !use_v2()) {
    if (T.claim && !T.sig2) T.claim = nullptr;  // dynamic claiming runs the two-SIG pipeline
    return launch_xgpu_ws(T, nullptr, 1, T.nparts, stream, err, mmax, kpmax, false);
  }
  return dispatch<false>(T, nullptr, 1, T.nparts, static_cast<cudaStream_t>(stream), err, mmax, kpmax, mom);
}

int launch_xgpu_emulated(XTask* tasks, int V, XTask* d_tasks, void* stream, std::string* err) {
  int mmax = 0, kpmax = 0, max_parts = 1;
  bool mom = false;
  for (int v = 0; v < V; ++v) {
    if (tasks[v].nparts == 0) continue;
    const int rc = check_task(tasks[v], &mmax, &kpmax, &mom, err);
    if (rc != RP_OK) return rc;
    max_parts = std::max(max_parts, static_cast<int>(tasks[v].nparts));
  }
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int v = 0; v < V; ++v) {
    tasks[v].nbuf = nbuf_setting();
    tasks[v].blag = blag_setting();
    tasks[v].sig2 = sig2_setting();
    tasks[v].lookahead = lookahead_setting();
    tasks[v].early_a = early_a_setting();
    if (tasks[v].claim && (!tasks[v].sig2 || mom || use_v2())) tasks[v].claim = nullptr;
  }
  const cudaError_t e = cudaMemcpyAsync(d_tasks, tasks, sizeof(XTask) * V, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    *err = std::string("xgpu emulation: task upload: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  if (!mom && !use_v2()) return launch_xgpu_ws(tasks[0], d_tasks, V, max_parts, stream, err, mmax, kpmax, true);
  // generic instantiations (KPM 8): emulation is a parity tool, not a timed path
  return dispatch<true>(tasks[0], d_tasks, V, max_parts, s, err, mmax, 8, mom);
}

}  // namespace rp
