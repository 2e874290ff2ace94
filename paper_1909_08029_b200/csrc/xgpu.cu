// Cross-GPU fused SGD + P-Reduce: this GPU's part of groups whose members span
// several GPUs of one NVSwitch node (one process per GPU, peer memory mapped
// through CUDA IPC). Push-based and pipelined chunk by chunk.
//
// alg1 step 4 for a group G on GPUs d_0 < ... < d_{kp-1} is one
// exchange step: a reduce-scatter + all-gather fused with the SGD of step 2
// and with the pre-reduction of co-resident members. The element range
// is cut into kp owner slices (tile-aligned float4 ranges; GPU d_i owns slice
// i) and every slice into nch chunks. Work items, in this order on every GPU:
//
//  A (o, c)  o != me: p = left fold over my local members of
//            y_m = fl(x_m - fl(lr_m g_m)) (ascending worker id) for chunk c of
//            slice o, STORED OVER NVLINK into owner o's staging buffer (row me),
//            then flag A[me][c] on owner o. By default each 256*U-float4 tile is
//            staged in shared memory and pushed by the TMA (cp.async.bulk).
//  B (c)     my slice: wait for A[d][c] from every peer d; own partial in
//            registers, peers' partials from my staging (local HBM); s = left
//            fold of the partials in ascending GPU id; xbar = fl(s / |G|)
//            (reading R1); store xbar into my local members and OVER NVLINK into
//            every peer's first local member ("x_first"), then flag B[me][c] on
//            every peer.
//  C (o, c)  o != me: wait for B[o][c]; xbar is already in my x_first; copy it
//            to my other local members (nothing to do for a lone member).
//
// No GPU ever reads peer memory: every NVLink byte is a store (bidirectional
// peer stores measured ~700 GB/s/direction vs ~660 for loads on B200,
// profiles/r01_nvlink_probe_2gpu.txt). NVLink bytes written per GPU:
// 2 (kp-1)/kp * 4N, the ring all-reduce bus bound; the transfers of chunk c
// overlap the compute of later chunks.
//
// Synchronization: 64-bit tags (unique per group) in per-GPU flag arrays
// (IPC-shared), written with st.release.sys after a system fence and polled
// with ld.acquire.sys. At kernel start each GPU posts READY to its peers; a GPU
// pushes partials into an owner's staging only after the owner's READY (the
// owner has finished its previous group, so the staging is free). The kernel
// ends when all of this GPU's inbound A and B flags have been seen, i.e. when
// no peer will write its memory for this group any more. The grid is at most
// the resident CTA count, so a CTA spinning on a flag never starves another.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "rp_internal.h"
#include "update.cuh"

namespace rp {

namespace {

constexpr int kXThreads = 256;
constexpr int64_t kTileF4 = static_cast<int64_t>(kXThreads) * 4;  // slice/chunk boundaries: multiples of every U

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

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 div4(float4 a, float k) {
  return make_float4(__fdiv_rn(a.x, k), __fdiv_rn(a.y, k), __fdiv_rn(a.z, k), __fdiv_rn(a.w, k));
}

// flag word of (slot, src GPU, kind, chunk) in a GPU's flag array
__device__ __forceinline__ unsigned long long* flag_at(unsigned long long* base, int slot, int src, int kind,
                                                       int64_t c) {
  return base + (static_cast<int64_t>(slot) * kFlagSrc + src) * kFlagStride +
         (kind == kFlagA ? c : (kind == kFlagB ? kMaxChunks + c : 2 * kMaxChunks));
}

// Watchdog: a peer that never posts its flag (a crashed rank, a broken collective contract)
// traps the kernel after kWaitTrapNs instead of spinning forever, so the process fails with a
// CUDA error rather than hanging the GPU. The clock is read once per 4096 polls.
constexpr unsigned long long kWaitTrapNs = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ void wait_flag(const unsigned long long* f, unsigned long long tag) {
  if (ld_acquire_sys(f) == tag) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (unsigned n = 1; ld_acquire_sys(f) != tag; ++n) {
    __nanosleep(32);
    if ((n & 4095u) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > kWaitTrapNs) __trap();
    }
  }
}

// ---- element access: fp32 replicas, or bf16 replicas with fp32 arithmetic (reading R26) ----
// A "vector" is 4 consecutive elements: 16 bytes of fp32 or 8 bytes of bf16. Staged partials
// are always fp32 (the fold runs in fp32); the mean is rounded once to bf16 when stored.
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t bf_rn(float v) {  // IEEE round-to-nearest-even (finite)
  const uint32_t b = __float_as_uint(v);
  return (b + 0x7fffu + ((b >> 16) & 1u)) >> 16;
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
__device__ __forceinline__ uint2 pack_bf4(float4 v) {
  return make_uint2(bf_rn(v.x) | (bf_rn(v.y) << 16), bf_rn(v.z) | (bf_rn(v.w) << 16));
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

// Local partial of my p.m (<= M) members at float4 index i (left fold, ascending worker id),
// with alg1 step 2 applied (and momentum buffers updated: each element's partial is
// computed exactly once, in its A or B item).
template <int M, bool MOM, bool BF = false>
__device__ __forceinline__ float4 local_partial4(const XPart& p, int64_t i) {
  float4 xv[M], gv[M], vv[MOM ? M : 1];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if (m < p.m) {
      xv[m] = ldx4<BF>(p.x[m], i);
      if (p.u[m].g) gv[m] = ldg4<BF>(p.u[m].g, i);
      if constexpr (MOM)
        if (p.u[m].v) vv[m] = ldv(p.u[m].v + 4 * i);
    }
  }
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if (m < p.m) {
      float4 vm = vv[MOM ? m : 0];
      const float4 y = step4<MOM>(xv[m], gv[m], vm, p.u[m]);
      if constexpr (MOM)
        if (p.u[m].v && p.u[m].g) stv(p.u[m].v + 4 * i, vm);
      s = m == 0 ? y : add4(s, y);
    }
  }
  return s;
}
template <int M, bool MOM, bool BF = false>
__device__ __forceinline__ float local_partial1(const XPart& p, int64_t j) {
  float s = step1x<MOM, BF>(p.x[0], p.u[0], j);
#pragma unroll
  for (int m = 1; m < M; ++m)
    if (m < p.m) s = __fadd_rn(s, step1x<MOM, BF>(p.x[m], p.u[m], j));
  return s;
}

// Chunk c of slice o: float4 range [lo, hi); the last chunk of the last slice also
// carries the n mod 4 scalar tail.
struct ChunkRange {
  int64_t lo, hi;
  bool tail;
};
__device__ __forceinline__ int64_t slice_lo(const XPart& p, int o) {
  return min(static_cast<int64_t>(o) * p.S4, p.n4);
}
__device__ __forceinline__ ChunkRange chunk_range(const XPart& p, int o, int64_t c) {
  const int64_t slo = slice_lo(p, o), shi = min(static_cast<int64_t>(o + 1) * p.S4, p.n4);
  ChunkRange r;
  r.lo = min(slo + c * p.CH, shi);
  r.hi = min(slo + (c + 1) * p.CH, shi);
  r.tail = (o == p.kp - 1) && (c == p.nch - 1) && p.rem > 0;
  return r;
}

// float offset of (row d, float4 index i relative to the slice start) in a staging
// region: row d holds the partials GPU d sends for the owner's slice; S4 + 1 float4
// per row so the tail scalars fit after the slice's float4 range.
__device__ __forceinline__ int64_t stage_off(const XPart& p, int d, int64_t i_rel) {
  return (static_cast<int64_t>(d) * (p.S4 + 1) + i_rel) * 4;
}

template <int M, int U, bool MOM>
__device__ void item_A(const XPart& p, int o, int64_t c) {
  const ChunkRange r = chunk_range(p, o, c);
  const int64_t slo = slice_lo(p, o);
  float* dst = p.stage[o];  // owner o's staging region (peer memory)
  for (int64_t t0 = r.lo; t0 < r.hi; t0 += kXThreads * U) {
    float4 s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < r.hi) s[u] = local_partial4<M, MOM>(p, i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < r.hi) stv(dst + stage_off(p, p.me, i - slo), s[u]);  // NVLink store
    }
  }
  if (r.tail && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    dst[stage_off(p, p.me, p.n4 - slo) + threadIdx.x] = local_partial1<M, MOM>(p, j);
  }
}

template <int M, int U, bool MOM, int KPM = kMaxXGpus>
__device__ void item_B(const XPart& p, int64_t c) {
  const int o = p.me;
  const ChunkRange r = chunk_range(p, o, c);
  const int64_t slo = slice_lo(p, o);
  const float* stage = p.stage[o];  // my staging region (local)
  const float kf = static_cast<float>(p.k_total);
  for (int64_t t0 = r.lo; t0 < r.hi; t0 += kXThreads * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < r.hi) {
        const float4 mine = local_partial4<M, MOM>(p, i);
        float4 part[KPM];
#pragma unroll
        for (int d = 0; d < KPM; ++d)
          if (d < p.kp && d != o) part[d] = ldv(stage + stage_off(p, d, i - slo));
        float4 s = o == 0 ? mine : part[0];
#pragma unroll
        for (int d = 1; d < KPM; ++d)
          if (d < p.kp) s = add4(s, d == o ? mine : part[d]);
        const float4 xbar = div4(s, kf);
#pragma unroll
        for (int m = 0; m < M; ++m)
          if (m < p.m) stv(p.x[m] + 4 * i, xbar);
#pragma unroll
        for (int d = 0; d < KPM; ++d)
          if (d < p.kp && d != o) stv(p.xfirst[d] + 4 * i, xbar);  // NVLink store
      }
    }
  }
  if (r.tail && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    const int64_t so = p.n4 - slo;
    const float mine = local_partial1<M, MOM>(p, j);
    float s = o == 0 ? mine : stage[stage_off(p, 0, so) + threadIdx.x];
    for (int d = 1; d < p.kp; ++d) s = __fadd_rn(s, d == o ? mine : stage[stage_off(p, d, so) + threadIdx.x]);
    const float xbar = __fdiv_rn(s, kf);
    for (int m = 0; m < p.m; ++m) p.x[m][j] = xbar;
    for (int d = 0; d < p.kp; ++d)
      if (d != o) p.xfirst[d][j] = xbar;
  }
}

// ---- TMA bulk-store variants of A and B (RP_XGPU_TMA=1) ---------------------------------
// The tile is staged in shared memory and one thread hands it to the Tensor Memory
// Accelerator (cp.async.bulk global <- shared::cta): one bulk transfer per 256*U float4
// instead of 256*U 16-byte peer stores; double-buffered; the flag follows
// cp.async.bulk.wait_group 0 + an async-proxy fence + a system fence.
__device__ __forceinline__ void bulk_store(void* dst_global, const void* src_smem, uint32_t bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(src_smem));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_global), "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }

template <int M, int U, bool MOM, bool BF = false>
__device__ void item_A_tma(const XPart& p, int o, int64_t c, float4* smem) {
  const ChunkRange r = chunk_range(p, o, c);
  const int64_t slo = slice_lo(p, o);
  float* dst = p.stage[o];
  constexpr int kTile = kXThreads * U;
  int buf = 0;
  for (int64_t t0 = r.lo; t0 < r.hi; t0 += kTile) {
    if (threadIdx.x == 0) bulk_wait_read1();  // the transfer issued two tiles ago has read `buf`
    __syncthreads();
    float4* sb = smem + buf * kTile;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < r.hi) sb[u * kXThreads + threadIdx.x] = local_partial4<M, MOM, BF>(p, i);
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t cnt = min(static_cast<int64_t>(kTile), r.hi - t0);
      bulk_store(dst + stage_off(p, p.me, t0 - slo), sb, static_cast<uint32_t>(cnt * 16));  // NVLink
      bulk_commit();
    }
    buf ^= 1;
  }
  if (r.tail && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    dst[stage_off(p, p.me, p.n4 - slo) + threadIdx.x] = local_partial1<M, MOM, BF>(p, j);
  }
  if (threadIdx.x == 0) {
    bulk_wait_all();
    fence_async_all();
  }
}

template <int M, int U, bool MOM, int KPM = kMaxXGpus, bool BF = false>
__device__ void item_B_tma(const XPart& p, int64_t c, float4* smem) {
  const int o = p.me;
  const ChunkRange r = chunk_range(p, o, c);
  const int64_t slo = slice_lo(p, o);
  const float* stage = p.stage[o];
  const float kf = static_cast<float>(p.k_total);
  constexpr int kTile = kXThreads * U;
  int buf = 0;
  for (int64_t t0 = r.lo; t0 < r.hi; t0 += kTile) {
    if (threadIdx.x == 0) bulk_wait_read1();
    __syncthreads();
    float4* sb = smem + buf * kTile;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < r.hi) {
        const float4 mine = local_partial4<M, MOM, BF>(p, i);
        float4 part[KPM];
#pragma unroll
        for (int d = 0; d < KPM; ++d)
          if (d < p.kp && d != o) part[d] = ldv(stage + stage_off(p, d, i - slo));
        float4 s = o == 0 ? mine : part[0];
#pragma unroll
        for (int d = 1; d < KPM; ++d)
          if (d < p.kp) s = add4(s, d == o ? mine : part[d]);
        const float4 xbar = div4(s, kf);
#pragma unroll
        for (int m = 0; m < M; ++m)
          if (m < p.m) stx4<BF>(p.x[m], i, xbar);
        if constexpr (BF) {
          reinterpret_cast<uint2*>(sb)[u * kXThreads + threadIdx.x] = pack_bf4(xbar);
          // bulk copies move multiples of 16 bytes: an odd last bf16 vector goes by plain store
          if (((r.hi - t0) & 1) && i == r.hi - 1 && r.hi - t0 <= kTile)
            for (int d = 0; d < KPM; ++d)
              if (d < p.kp && d != o) stx4<true>(p.xfirst[d], i, xbar);  // NVLink
        } else {
          sb[u * kXThreads + threadIdx.x] = xbar;
        }
      }
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t cnt = min(static_cast<int64_t>(kTile), r.hi - t0);
      const uint32_t bytes = static_cast<uint32_t>(BF ? (cnt & ~1LL) * 8 : cnt * 16);
      for (int d = 0; d < p.kp; ++d)
        if (d != o) {
          void* dst = BF ? static_cast<void*>(reinterpret_cast<uint16_t*>(p.xfirst[d]) + 4 * t0)
                         : static_cast<void*>(p.xfirst[d] + 4 * t0);
          if (bytes) bulk_store(dst, sb, bytes);  // NVLink
        }
      bulk_commit();
    }
    buf ^= 1;
  }
  if (r.tail && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    const int64_t so = p.n4 - slo;
    const float mine = local_partial1<M, MOM, BF>(p, j);
    float s = o == 0 ? mine : stage[stage_off(p, 0, so) + threadIdx.x];
    for (int d = 1; d < p.kp; ++d) s = __fadd_rn(s, d == o ? mine : stage[stage_off(p, d, so) + threadIdx.x]);
    const float xbar = __fdiv_rn(s, kf);
    for (int m = 0; m < p.m; ++m) stx1<BF>(p.x[m], j, xbar);
    for (int d = 0; d < p.kp; ++d)
      if (d != o) stx1<BF>(p.xfirst[d], j, xbar);
  }
  if (threadIdx.x == 0) {
    bulk_wait_all();
    fence_async_all();
  }
}

template <int M, int U, bool BF = false>
__device__ void item_C(const XPart& p, int o, int64_t c) {
  if (p.m == 1) return;  // the owner stored xbar straight into my only replica
  const ChunkRange r = chunk_range(p, o, c);
  for (int64_t t0 = r.lo; t0 < r.hi; t0 += kXThreads * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < r.hi) v[u] = ldx4<BF>(p.x[0], i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < r.hi) {
#pragma unroll
        for (int m = 1; m < M; ++m)
          if (m < p.m) stx4<BF>(p.x[m], i, v[u]);  // exact for bf16 (already rounded)
      }
    }
  }
  if (r.tail && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    const float v = ldx1<BF>(p.x[0], j);
    for (int m = 1; m < p.m; ++m) stx1<BF>(p.x[m], j, v);
  }
}

// L item: chunk c of fused intra-GPU group gi (alg1 steps 2+4 on one GPU, pinned fold)
template <int K, int U, bool MOM>
__device__ void item_L_k(const XLocalGroup& G, int64_t lo, int64_t hi, bool tail, int64_t n4, int rem) {
  for (int64_t t0 = lo; t0 < hi; t0 += kXThreads * U) {
    float4 xv[U][K], gv[U][K], vv[U][MOM ? K : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < hi)
#pragma unroll
        for (int m = 0; m < K; ++m) {
          xv[u][m] = ldv(G.x[m] + 4 * i);
          if (G.u[m].g) gv[u][m] = ldg_nc(G.u[m].g + 4 * i);
          if constexpr (MOM)
            if (G.u[m].v) vv[u][m] = ldv(G.u[m].v + 4 * i);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = t0 + u * kXThreads + threadIdx.x;
      if (i < hi) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int m = 0; m < K; ++m) {
          float4 vm = vv[u][MOM ? m : 0];
          const float4 y = step4<MOM>(xv[u][m], gv[u][m], vm, G.u[m]);
          if constexpr (MOM)
            if (G.u[m].v && G.u[m].g) stv(G.u[m].v + 4 * i, vm);
          s = m == 0 ? y : add4(s, y);
        }
        if (K > 1) s = div4(s, static_cast<float>(K));
#pragma unroll
        for (int m = 0; m < K; ++m) stv(G.x[m] + 4 * i, s);
      }
    }
  }
  if (tail && threadIdx.x < rem) {
    const int64_t j = 4 * n4 + threadIdx.x;
    float s = step1<MOM>(G.x[0][j], G.u[0], j);
    for (int m = 1; m < K; ++m) s = __fadd_rn(s, step1<MOM>(G.x[m][j], G.u[m], j));
    if (K > 1) s = __fdiv_rn(s, static_cast<float>(K));
    for (int m = 0; m < K; ++m) G.x[m][j] = s;
  }
}

template <int U, bool MOM>
__device__ void item_L(const XTask& T, int64_t idx) {
  const XLocalGroup& G = T.lg[idx / T.nchl];
  const int64_t c = idx % T.nchl;
  const int64_t n4 = T.n / 4;
  const int rem = static_cast<int>(T.n - 4 * n4);
  const int64_t lo = min(c * T.chl, n4), hi = min((c + 1) * T.chl, n4);
  const bool tail = (c == T.nchl - 1) && rem > 0;
  switch (G.k) {
    case 1: item_L_k<1, U, MOM>(G, lo, hi, tail, n4, rem); break;
    case 2: item_L_k<2, U, MOM>(G, lo, hi, tail, n4, rem); break;
    case 3: item_L_k<3, U, MOM>(G, lo, hi, tail, n4, rem); break;
    default: item_L_k<4, U, MOM>(G, lo, hi, tail, n4, rem); break;
  }
}

// item index within an A or C range of part p -> (slice o != me, chunk c), chunk-major
__device__ __forceinline__ void other_item(const XPart& p, int64_t i, int* o, int64_t* c) {
  const int j = static_cast<int>(i % (p.kp - 1));
  *c = i / (p.kp - 1);
  *o = j < p.me ? j : j + 1;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// M bounds the local member count of every part (register budget).
template <int M, int U, bool MOM, bool TMA, int MINB = 2, int KPM = kMaxXGpus, bool BF = false>
__global__ void __launch_bounds__(kXThreads, MINB) xgpu_kernel(const XTask T) {
  static_assert(!BF || (TMA && !MOM), "bf16 replicas: TMA variants, plain SGD only");
  extern __shared__ float4 xsmem[];  // TMA: two tiles of kXThreads * U float4
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // READY: my staging is free for these groups (my previous kernel has finished)
    for (int pi = 0; pi < T.nparts; ++pi) {
      const XPart& p = T.part[pi];
      for (int d = 0; d < p.kp; ++d)
        if (d != p.me) st_release_sys(flag_at(p.pflags[d], p.slot, T.my_gpu, kFlagReady, 0), p.tag);
    }
  }
  uint32_t ready_seen = 0;  // bit 8*pi + o: READY of part pi's owner o observed (thread 0)
  for (int64_t q = blockIdx.x; q < T.total_items; q += gridDim.x) {
    const uint32_t it = T.items[q];
    const int region = static_cast<int>(it >> 30);  // 0 = A, 1 = B, 2 = C, 3 = L
    const int pi = static_cast<int>((it >> 27) & 7);
    int64_t t = static_cast<int64_t>(it & ((1u << 27) - 1));
    unsigned long long ts = 0, tr = 0;
    if (T.prof && threadIdx.x == 0) ts = gtimer();
    if (region == 3) {
      if (T.prof && threadIdx.x == 0) tr = gtimer();
      if constexpr (!BF) item_L<1, MOM>(T, t);  // bf16 launches carry no L items (launch_xgpu)
      if (T.prof) {
        __syncthreads();
        if (threadIdx.x == 0) {
          XItemRecord rec{ts, tr, gtimer(),
                          (3ull << 62) | (static_cast<unsigned long long>(blockIdx.x & 0xFFFFFF) << 32) |
                              static_cast<unsigned long long>(t)};
          T.prof[q] = rec;
        }
      }
      continue;
    }
    const XPart& p = T.part[pi];
    if (region == 0) {
      int o;
      int64_t c;
      other_item(p, t, &o, &c);
      const uint32_t bit = 1u << (8 * (pi & 3) + o);
      if (threadIdx.x == 0 && (pi >= 4 || !(ready_seen & bit))) {
        wait_flag(flag_at(T.my_flags, p.slot, p.gpu[o], kFlagReady, 0), p.tag);
        if (pi < 4) ready_seen |= bit;
      }
      __syncthreads();
      if (T.prof && threadIdx.x == 0) tr = gtimer();
      if constexpr (TMA)
        item_A_tma<M, U, MOM, BF>(p, o, c, xsmem);
      else
        item_A<M, U, MOM>(p, o, c);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        st_release_sys(flag_at(p.pflags[o], p.slot, T.my_gpu, kFlagA, c), p.tag);
      }
    } else if (region == 1) {
      if (threadIdx.x == 0)
        for (int d = 0; d < p.kp; ++d)
          if (d != p.me) wait_flag(flag_at(T.my_flags, p.slot, p.gpu[d], kFlagA, t), p.tag);
      __syncthreads();
      if (T.prof && threadIdx.x == 0) tr = gtimer();
      if constexpr (TMA)
        item_B_tma<M, U, MOM, KPM, BF>(p, t, xsmem);
      else
        item_B<M, 1, MOM, KPM>(p, t);  // B keeps M + kp - 1 loads per float4 in flight already
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        for (int d = 0; d < p.kp; ++d)
          if (d != p.me) st_release_sys(flag_at(p.pflags[d], p.slot, T.my_gpu, kFlagB, t), p.tag);
      }
    } else {
      int o;
      int64_t c;
      other_item(p, t, &o, &c);
      if (threadIdx.x == 0) wait_flag(flag_at(T.my_flags, p.slot, p.gpu[o], kFlagB, c), p.tag);
      __syncthreads();
      if (T.prof && threadIdx.x == 0) tr = gtimer();
      item_C<M, U, BF>(p, o, c);
    }
    __syncthreads();
    if (T.prof && threadIdx.x == 0) {
      XItemRecord rec;
      rec.t_start = ts;
      rec.t_ready = tr;
      rec.t_end = gtimer();
      rec.meta = (static_cast<unsigned long long>(region) << 62) | (static_cast<unsigned long long>(pi) << 56) |
                 (static_cast<unsigned long long>(blockIdx.x & 0xFFFFFF) << 32) | static_cast<unsigned long long>(t);
      T.prof[q] = rec;
    }
  }
}

int g_sms = 0;

// Tuning knobs (read once): RP_XGPU_U (1|2|4 float4 per thread and tile row),
// RP_XGPU_CTAS_PER_SM (cap on resident CTAs used), RP_XGPU_CHUNK_F4 (min chunk).
int env_int(const char* name, int def) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : def;
}
int g_u = -1, g_cps = -1, g_lag = -1, g_order = -1, g_tma = -1, g_lean = -1;
int64_t g_min_chunk = -1;

// Host-built work-item order, cached per launch shape. Virtual time in units of a
// part's chunks: A(o, c) at c, B(c) at c + lag, C(o, c) at c + 2 lag; L items spread
// evenly over the A and B items. The default lag = nch runs all A items, then all B
// items (chunk-pipelined lags were slower on 2 B200: more, smaller chunks pay more
// system fences; profiles/r01_xgpu_lag_sweep_2gpu.txt).
int item_list(const XTask& T, int64_t ctas, const uint32_t** out, int64_t* count, std::string* err) {
  static std::mutex mu;
  static std::map<std::string, std::pair<uint32_t*, int64_t>> cache;
  std::string key = std::to_string(g_order) + "/" + std::to_string(T.my_gpu) + "/" + std::to_string(ctas) + "/" + std::to_string(T.nlocal) + "/" +
                    std::to_string(T.nchl);
  for (int pi = 0; pi < T.nparts; ++pi)
    key += "/" + std::to_string(T.part[pi].kp) + "," + std::to_string(T.part[pi].me) + "," +
           std::to_string(T.part[pi].nch);
  std::lock_guard<std::mutex> lk(mu);
  auto hit = cache.find(key);
  if (hit != cache.end()) {
    *out = hit->second.first;
    *count = hit->second.second;
    return RP_OK;
  }
  struct Ent {
    double t;
    int order;
    uint32_t code;
  };
  std::vector<Ent> v;
  double tmax = 1.0;
  for (int pi = 0; pi < T.nparts; ++pi) {
    const XPart& p = T.part[pi];
    const double nch = static_cast<double>(p.nch);
    // lag: RP_XGPU_LAG (chunks) or, by default, all A items before any B item
    const double lag = g_lag > 0 ? std::min<double>(nch, g_lag) : nch;
    const uint32_t P = static_cast<uint32_t>(pi) << 27;
    for (int64_t i = 0; i < (p.kp - 1) * p.nch; ++i) {
      const double c = static_cast<double>(i / (p.kp - 1));
      v.push_back({c / nch, 0, (0u << 30) | P | static_cast<uint32_t>(i)});
      v.push_back({(c + 2 * lag) / nch, 2, (2u << 30) | P | static_cast<uint32_t>(i)});
    }
    for (int64_t c = 0; c < p.nch; ++c) v.push_back({(c + lag) / nch, 1, (1u << 30) | P | static_cast<uint32_t>(c)});
    tmax = std::max(tmax, (nch + lag) / nch);
  }
  const int64_t nl = static_cast<int64_t>(T.nlocal) * T.nchl;
  for (int64_t l = 0; l < nl; ++l) v.push_back({tmax * static_cast<double>(l) / nl, 3, (3u << 30) | static_cast<uint32_t>(l)});
  std::stable_sort(v.begin(), v.end(), [](const Ent& a, const Ent& b) { return a.t < b.t || (a.t == b.t && a.order < b.order); });
  std::vector<uint32_t> h(v.size());
  for (size_t i = 0; i < v.size(); ++i) h[i] = v[i].code;
  if (g_order == 1) {
    // role split: even grid slots take A/L items, odd slots B items (both in chunk order), so
    // B(c) starts as soon as the peers' A(c) lands; C items last
    std::vector<uint32_t> ab, bb, cc;
    for (uint32_t x : h) ((x >> 30) == 1 ? bb : ((x >> 30) == 2 ? cc : ab)).push_back(x);
    h.clear();
    size_t ia = 0, ib = 0;
    while (ia < ab.size() || ib < bb.size()) {
      const bool slot_b = (h.size() % 2) == 1;
      if ((slot_b && ib < bb.size()) || ia >= ab.size())
        h.push_back(bb[ib++]);
      else
        h.push_back(ab[ia++]);
    }
    h.insert(h.end(), cc.begin(), cc.end());
  }
  uint32_t* d = nullptr;
  if (cudaMalloc(&d, h.size() * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemcpy(d, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    *err = "xgpu: item list upload failed";
    return RP_ECUDA;
  }
  cache[key] = {d, static_cast<int64_t>(h.size())};
  *out = d;
  *count = static_cast<int64_t>(h.size());
  return RP_OK;
}


template <int M, int U, bool MOM = false, bool TMA = false, int MINB = 2, int KPM = kMaxXGpus, bool BF = false>
int launch_m(XTask& T, cudaStream_t stream, std::string* err) {
  static int occ = 0;
  const size_t smem = TMA ? 2 * sizeof(float4) * kXThreads * U : 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, xgpu_kernel<M, U, MOM, TMA, MINB, KPM, BF>, kXThreads, smem) !=
            cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  int64_t cap = static_cast<int64_t>(g_sms) * occ;  // all CTAs co-resident
  if (g_cps > 0) cap = std::min<int64_t>(cap, static_cast<int64_t>(g_sms) * g_cps);
  const int64_t grid_cap = T.max_ctas > 0 ? std::min<int64_t>(cap, T.max_ctas) : cap;
  // chunk geometry depends on the SM count only, never on this launch's grid or
  // instantiation: every GPU of a group must cut the same chunks (flags are per chunk)
  const int64_t geom = static_cast<int64_t>(g_sms) * 2;
  if (g_min_chunk < 0) g_min_chunk = env_int("RP_XGPU_CHUNK_F4", static_cast<int>(kMinChunkF4));
  for (int pi = 0; pi < T.nparts; ++pi) {
    XPart& p = T.part[pi];
    // chunk: about one A and one B item per resident CTA (each CTA pays the system fence
    // behind a flag about twice per group: measured best on 2 B200, profiles/r01_xgpu_*),
    // at least g_min_chunk float4, at most kMaxChunks chunks per slice
    int64_t ch = std::max<int64_t>({(p.S4 + geom - 1) / geom, g_min_chunk, (p.S4 + kMaxChunks - 1) / kMaxChunks});
    p.CH = (ch + kTileF4 - 1) / kTileF4 * kTileF4;
    p.nch = std::max<int64_t>(1, (p.S4 + p.CH - 1) / p.CH);
  }
  const int64_t n4 = T.n / 4;
  T.chl = std::max<int64_t>(kTileF4, (std::max<int64_t>(n4, 1) * T.nlocal / std::max<int64_t>(cap, 1) + kTileF4 - 1) /
                                         kTileF4 * kTileF4);
  T.chl = std::max<int64_t>(T.chl, g_min_chunk / kTileF4 * kTileF4);
  T.nchl = std::max<int64_t>(1, (n4 + T.chl - 1) / T.chl);
  const int rc = item_list(T, cap, &T.items, &T.total_items, err);
  if (rc != RP_OK) return rc;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min(grid_cap, T.total_items)));
  xgpu_kernel<M, U, MOM, TMA, MINB, KPM, BF><<<blocks, kXThreads, smem, stream>>>(T);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("xgpu kernel launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

}  // namespace

void xgpu_geometry(XPart& p, int64_t n) {
  p.n4 = n / 4;
  p.rem = static_cast<int32_t>(n - 4 * p.n4);
  p.S4 = ((p.n4 + p.kp - 1) / p.kp + kTileF4 - 1) / kTileF4 * kTileF4;
  p.CH = std::max<int64_t>(p.S4, kTileF4);  // chunking is chosen by the launcher
  p.nch = 1;
}

int64_t xgpu_stage_region_bytes(int64_t n) {
  // kp rows of (S4 + 1) float4, S4 <= n4/kp + tile: at most 4n + 16 * kp * (tile + 2)
  return 4 * n + 16LL * kMaxXGpus * (kTileF4 + 2);
}

int launch_xgpu(XTask& T, void* stream, std::string* err) {
  if (T.nparts < 1 || T.nparts > kMaxXParts || T.nlocal < 0 || T.nlocal > kMaxXLocalGroups) {
    *err = "xgpu: bad part count";
    return RP_EINVAL;
  }
  for (int gi = 0; gi < T.nlocal; ++gi) {
    const XLocalGroup& G = T.lg[gi];
    if (G.k < 1 || G.k > kMaxFusedK) {
      *err = "xgpu: fused local groups must have 1..4 members";
      return RP_EINVAL;
    }
    for (int m = 0; m < G.k; ++m)
      if (!G.x[m] || (reinterpret_cast<uintptr_t>(G.x[m]) & 15) || (reinterpret_cast<uintptr_t>(G.u[m].g) & 15) ||
          (reinterpret_cast<uintptr_t>(G.u[m].v) & 15)) {
        *err = "xgpu: local replica / gradient pointers must be non-null and 16-byte aligned";
        return RP_EINVAL;
      }
  }
  int mmax = 0;
  for (int pi = 0; pi < T.nparts; ++pi) {
    const XPart& p = T.part[pi];
    if (p.m < 1 || p.m > kMaxXLocal || p.kp < 2 || p.kp > kMaxXGpus || p.me < 0 || p.me >= p.kp) {
      *err = "xgpu: bad part descriptor";
      return RP_EINVAL;
    }
    for (int d = 0; d < p.kp; ++d)
      if (!p.stage[d] || !p.xfirst[d] || !p.pflags[d] || (reinterpret_cast<uintptr_t>(p.xfirst[d]) & 15) ||
          (reinterpret_cast<uintptr_t>(p.stage[d]) & 15)) {
        *err = "xgpu: peer pointers missing (call rp_peer_import) or misaligned";
        return RP_EINVAL;
      }
    mmax = std::max(mmax, p.m);
  }
  // every cross part of a step is in ONE launch (two launches on one stream could
  // wait on each other across GPUs), so M is the largest local member count
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  bool mom = false;
  for (int pi = 0; pi < T.nparts; ++pi)
    for (int m = 0; m < T.part[pi].m; ++m) mom = mom || (T.part[pi].u[m].v && T.part[pi].u[m].g);
  for (int gi = 0; gi < T.nlocal; ++gi)
    for (int m = 0; m < T.lg[gi].k; ++m) mom = mom || (T.lg[gi].u[m].v && T.lg[gi].u[m].g);
  if (g_u < 0) {
    g_u = env_int("RP_XGPU_U", 4);
    g_cps = env_int("RP_XGPU_CTAS_PER_SM", 0);
    g_lag = env_int("RP_XGPU_LAG", 0);
    g_order = env_int("RP_XGPU_ORDER", 0);
    g_tma = env_int("RP_XGPU_TMA", 1);
    g_lean = env_int("RP_XGPU_LEAN", 0);
  }
  if (T.bf16) {  // bf16 replicas (reading R26): TMA pushes, plain SGD, no fused local groups
    if (mom || T.nlocal > 0) {
      *err = "xgpu: bf16 replicas take plain SGD and no fused local groups";
      return RP_EINVAL;
    }
    if (mmax <= 1) return launch_m<1, 2, false, true, 2, kMaxXGpus, true>(T, s, err);
    if (mmax <= 2) return launch_m<2, 2, false, true, 2, kMaxXGpus, true>(T, s, err);
    if (mmax <= 4) return launch_m<4, 1, false, true, 2, kMaxXGpus, true>(T, s, err);
    return launch_m<8, 1, false, true, 2, kMaxXGpus, true>(T, s, err);
  }
  if (mom) {  // momentum buffers: separate instantiations keep the plain path's registers
    if (g_tma > 0) {
      if (mmax <= 1) return launch_m<1, 1, true, true>(T, s, err);
      if (mmax <= 2) return launch_m<2, 1, true, true>(T, s, err);
      if (mmax <= 4) return launch_m<4, 1, true, true>(T, s, err);
      return launch_m<8, 1, true, true>(T, s, err);
    }
    if (mmax <= 1) return launch_m<1, 1, true>(T, s, err);
    if (mmax <= 2) return launch_m<2, 1, true>(T, s, err);
    if (mmax <= 4) return launch_m<4, 1, true>(T, s, err);
    return launch_m<8, 1, true>(T, s, err);
  }
  // RP_XGPU_LEAN=1 (experiment, off by default: no gain measured, profiles/r01_split/
  // sweep_4_lean.txt): beside an intra-GPU launch, a lean instantiation (<= 80 registers at
  // 3 CTAs per SM) so the intra-GPU kernel's CTAs still fit on every SM next to it
  int kpmax = 0;
  for (int pi = 0; pi < T.nparts; ++pi) kpmax = std::max(kpmax, T.part[pi].kp);
  if (T.max_ctas > 0 && g_tma > 0 && mmax <= 2 && kpmax <= 4 && g_lean != 0)
    return mmax <= 1 ? launch_m<1, 1, false, true, 3, 4>(T, s, err) : launch_m<2, 1, false, true, 3, 4>(T, s, err);
  if (g_tma > 0) {  // default: TMA bulk stores for the NVLink pushes (+17-31 % on 2 B200,
                    // profiles/r01_xgpu_tma_sweep_2gpu.txt); RP_XGPU_TMA=0 selects peer STG.128
    if (mmax <= 1) return g_u >= 4 ? launch_m<1, 4, false, true>(T, s, err) : launch_m<1, 2, false, true>(T, s, err);
    if (mmax <= 2) return launch_m<2, 2, false, true>(T, s, err);
    if (mmax <= 4) return launch_m<4, 1, false, true>(T, s, err);
    return launch_m<8, 1, false, true>(T, s, err);
  }
  if (mmax <= 1) return g_u >= 4 ? launch_m<1, 4>(T, s, err) : (g_u == 1 ? launch_m<1, 1>(T, s, err) : launch_m<1, 2>(T, s, err));
  if (mmax <= 2) return g_u == 1 ? launch_m<2, 1>(T, s, err) : launch_m<2, 2>(T, s, err);  // U=4 spills
  if (mmax <= 4) return launch_m<4, 1>(T, s, err);
  return launch_m<8, 1>(T, s, err);
}

}  // namespace rp
