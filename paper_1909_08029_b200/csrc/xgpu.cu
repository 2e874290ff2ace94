// Cross-GPU fused SGD + P-Reduce: this GPU's part of groups whose members span
// several GPUs of one NVSwitch node (one process per GPU, peer memory mapped
// through CUDA IPC).
//
// alg1 step 4 for a group G on GPUs d_0 < ... < d_{kp-1} is one
// exchange step: a reduce-scatter + all-gather fused with the SGD of step 2
// and with the pre-reduction of co-resident members. The element range
// is cut into kp owner slices (tile-aligned float4 ranges); GPU d_i owns slice i.
//
//  A (HBM only)   for every slice o != mine: p_me = left fold over my local
//                 members of y_m = fl(x_m - fl(lr_m g_m)) (ascending worker id),
//                 stored in place into my first local member's replica
//                 ("x_first"; the replicas are scratch while the group is in
//                 flight). Then signal A-done to every peer.
//  B (NVLink in)  for my slice: p_me in registers; for every other GPU d, wait
//                 for its A-done and load its partial from its x_first over
//                 NVLink; s = left fold of the partials in ascending GPU id;
//                 xbar = fl(s / |G|) (reading R1); store xbar into all my local
//                 members. Signal B-done.
//  C (NVLink in)  for every slice o != mine: wait for owner o's B-done, load
//                 xbar from o's x_first, store into all my local members.
//                 Signal C-done once all my B and C tiles (every peer read) are
//                 finished; the kernel ends only after every peer's C-done
//                 (nobody may touch a replica a peer still reads).
// NVLink bytes read per GPU: 2 (kp-1)/kp * 4N, the ring all-reduce bus bound.
//
// Synchronization: 64-bit tags in a per-GPU flag array (IPC-shared), written
// by peers with st.release.sys and polled with ld.acquire.sys. Each CTA adds
// its finished tiles of a phase to a local counter once (after a gpu-scope
// fence); the CTA completing the phase issues a system fence and writes the
// tag into every peer's flag array. The grid is at most the resident CTA count
// so a CTA spinning on a flag never starves another CTA of this kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "rp_internal.h"

namespace rp {

namespace {

constexpr int kXThreads = 256;

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

__device__ __forceinline__ float sgd1(float x, float g, float lr) { return __fsub_rn(x, __fmul_rn(lr, g)); }
__device__ __forceinline__ float4 sgd4(float4 x, float4 g, float lr) {
  return make_float4(sgd1(x.x, g.x, lr), sgd1(x.y, g.y, lr), sgd1(x.z, g.z, lr), sgd1(x.w, g.w, lr));
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 div4(float4 a, float k) {
  return make_float4(__fdiv_rn(a.x, k), __fdiv_rn(a.y, k), __fdiv_rn(a.z, k), __fdiv_rn(a.w, k));
}

__device__ __forceinline__ unsigned long long* flag_at(unsigned long long* base, int slot, int src, int phase) {
  return base + (static_cast<int64_t>(slot) * kFlagSrc + src) * kFlagPhases + phase;
}

// Geometry of part p: slice o is float4 range [o*S4, min((o+1)*S4, n4)); tiles of
// kXThreads*U float4. The last slice also carries the n mod 4 scalar tail, which
// gets an extra tile when the last regular tile is full (or the slice is empty).
template <int U>
struct Geo {
  int64_t n4, S4;
  int rem, kp;
  __device__ __forceinline__ int64_t lo(int o) const { return min(static_cast<int64_t>(o) * S4, n4); }
  __device__ __forceinline__ int64_t hi(int o) const { return min(static_cast<int64_t>(o + 1) * S4, n4); }
  __device__ __forceinline__ int64_t tiles(int o) const {
    const int64_t len = hi(o) - lo(o);
    int64_t t = (len + kXThreads * U - 1) / (kXThreads * U);
    if (o == kp - 1 && rem > 0 && len % (kXThreads * U) == 0) ++t;
    return t;
  }
};

// Local partial of my p.m (<= M) members at float4 index i (left fold, ascending worker id).
template <int M>
__device__ __forceinline__ float4 local_partial4(const XPart& p, int64_t i) {
  float4 xv[M], gv[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if (m < p.m) {
      xv[m] = ldv(p.x[m] + 4 * i);
      if (p.g[m]) gv[m] = ldg_nc(p.g[m] + 4 * i);
    }
  }
  float4 s = p.g[0] ? sgd4(xv[0], gv[0], p.lr[0]) : xv[0];
#pragma unroll
  for (int m = 1; m < M; ++m)
    if (m < p.m) s = add4(s, p.g[m] ? sgd4(xv[m], gv[m], p.lr[m]) : xv[m]);
  return s;
}
template <int M>
__device__ __forceinline__ float local_partial1(const XPart& p, int64_t j) {
  float s = p.g[0] ? sgd1(p.x[0][j], p.g[0][j], p.lr[0]) : p.x[0][j];
#pragma unroll
  for (int m = 1; m < M; ++m)
    if (m < p.m) s = __fadd_rn(s, p.g[m] ? sgd1(p.x[m][j], p.g[m][j], p.lr[m]) : p.x[m][j]);
  return s;
}

__device__ __forceinline__ bool needs_partial_store(const XPart& p) {
  return p.m > 1 || p.g[0] != nullptr;  // a lone member without a staged step: partial == x
}

template <int M>
__device__ __forceinline__ void store_members4(const XPart& p, int64_t i, float4 v) {
#pragma unroll
  for (int m = 0; m < M; ++m)
    if (m < p.m) stv(p.x[m] + 4 * i, v);
}
template <int M>
__device__ __forceinline__ void store_members1(const XPart& p, int64_t j, float v) {
#pragma unroll
  for (int m = 0; m < M; ++m)
    if (m < p.m) p.x[m][j] = v;
}

// ---- phase bodies over one tile ----------------------------------------------------------
template <int M, int U>
__device__ void tile_A(const XPart& p, const Geo<U>& geo, int o, int64_t t) {
  const int64_t lo = geo.lo(o), hi = geo.hi(o);
  const int64_t i0 = lo + t * kXThreads * U;
  const bool store = needs_partial_store(p);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * kXThreads + threadIdx.x;
    if (i < hi) {
      const float4 s = local_partial4<M>(p, i);
      if (store) stv(p.x[0] + 4 * i, s);
    }
  }
  if (o == geo.kp - 1 && t == geo.tiles(o) - 1 && threadIdx.x < geo.rem) {
    const int64_t j = 4 * geo.n4 + threadIdx.x;
    const float s = local_partial1<M>(p, j);
    if (store) p.x[0][j] = s;
  }
}

template <int M, int U>
__device__ void tile_B(const XPart& p, const Geo<U>& geo, int64_t t) {
  const int o = p.me;
  const int64_t lo = geo.lo(o), hi = geo.hi(o);
  const int64_t i0 = lo + t * kXThreads * U;
  const float kf = static_cast<float>(p.k_total);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * kXThreads + threadIdx.x;
    if (i < hi) {
      const float4 mine = local_partial4<M>(p, i);
      float4 part[kMaxXGpus];
#pragma unroll
      for (int d = 0; d < kMaxXGpus; ++d)
        if (d < p.kp && d != p.me) part[d] = ldv(p.src[d] + 4 * i);  // NVLink
      float4 s = p.me == 0 ? mine : part[0];
#pragma unroll
      for (int d = 1; d < kMaxXGpus; ++d)
        if (d < p.kp) s = add4(s, d == p.me ? mine : part[d]);
      store_members4<M>(p, i, div4(s, kf));
    }
  }
  if (o == geo.kp - 1 && t == geo.tiles(o) - 1 && threadIdx.x < geo.rem) {
    const int64_t j = 4 * geo.n4 + threadIdx.x;
    const float mine = local_partial1<M>(p, j);
    float s = p.me == 0 ? mine : p.src[0][j];
    for (int d = 1; d < p.kp; ++d) s = __fadd_rn(s, d == p.me ? mine : p.src[d][j]);
    store_members1<M>(p, j, __fdiv_rn(s, kf));
  }
}

template <int M, int U>
__device__ void tile_C(const XPart& p, const Geo<U>& geo, int o, int64_t t) {
  const int64_t lo = geo.lo(o), hi = geo.hi(o);
  const int64_t i0 = lo + t * kXThreads * U;
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * kXThreads + threadIdx.x;
    if (i < hi) v[u] = ldv(p.src[o] + 4 * i);  // NVLink
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * kXThreads + threadIdx.x;
    if (i < hi) store_members4<M>(p, i, v[u]);
  }
  if (o == geo.kp - 1 && t == geo.tiles(o) - 1 && threadIdx.x < geo.rem) {
    const int64_t j = 4 * geo.n4 + threadIdx.x;
    store_members1<M>(p, j, p.src[o][j]);
  }
}

// Map the t-th tile of part p's A (or C) range to (slice o != me, tile within slice).
template <int U>
__device__ __forceinline__ void other_slice_tile(const XPart& p, const Geo<U>& geo, int64_t t, int* o_out,
                                                 int64_t* t_out) {
  for (int o = 0; o < p.kp; ++o) {
    if (o == p.me) continue;
    const int64_t n = geo.tiles(o);
    if (t < n) {
      *o_out = o;
      *t_out = t;
      return;
    }
    t -= n;
  }
  *o_out = -1;
  *t_out = 0;
}

__device__ void signal_peers(const XTask& T, const XPart& p, int phase) {
  __threadfence_system();
  for (int d = 0; d < p.kp; ++d)
    if (d != p.me) st_release_sys(flag_at(p.pflags[d], p.slot, T.my_gpu, phase), p.tag);
}

__device__ void wait_peer(const XTask& T, const XPart& p, int d, int phase) {
  const unsigned long long* f = flag_at(T.my_flags, p.slot, p.gpu[d], phase);
  while (ld_acquire_sys(f) != p.tag) __nanosleep(64);
}

// Add this CTA's finished tiles of (part, phase) to the phase counter; the CTA
// that completes the phase signals every peer.
__device__ void flush_count(const XTask& T, int pi, int phase, int64_t mine, int64_t total) {
  if (mine == 0) return;
  const XPart& p = T.part[pi];
  __threadfence();
  unsigned long long* c = T.my_counters + static_cast<int64_t>(p.slot) * kFlagPhases + phase;
  const unsigned long long before = atomicAdd(c, static_cast<unsigned long long>(mine));
  if (before + mine == static_cast<unsigned long long>(total)) {
    atomicExch(c, 0ull);
    signal_peers(T, p, phase);
  }
}

// Counters per part: A tiles -> A-done ("my partials are ready"); B tiles -> B-done
// ("my slice's means are ready"); B and C tiles -> C-done ("I have finished
// reading every peer's memory for this group"), the condition for peers to end.
__device__ void publish(const XTask& T, int region, const int64_t* cnt) {
  for (int pi = 0; pi < T.nparts; ++pi) {
    const XPart& p = T.part[pi];
    if (region == 0) {
      flush_count(T, pi, kPhaseA, cnt[pi], p.ta);
    } else {
      if (region == 1) flush_count(T, pi, kPhaseB, cnt[pi], p.tb);
      flush_count(T, pi, kPhaseC, cnt[pi], p.tb + p.ta);
    }
  }
}

// M bounds the local member count of every part (register budget).
template <int M, int U>
__global__ void __launch_bounds__(kXThreads) xgpu_kernel(const XTask T) {
  // Phases with no tiles anywhere are complete from the start.
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int pi = 0; pi < T.nparts; ++pi) {
      const XPart& p = T.part[pi];
      if (p.ta == 0) signal_peers(T, p, kPhaseA);
      if (p.tb == 0) signal_peers(T, p, kPhaseB);
      // C-done needs B + C tiles, and ta + tb >= 1 whenever n >= 1
    }
  }
  int64_t cnt[kMaxXParts];
  uint32_t confirmed[kMaxXParts];  // bit d: A-done of GPU index d seen; bit 8+o: B-done of owner o seen
#pragma unroll
  for (int pi = 0; pi < kMaxXParts; ++pi) {
    cnt[pi] = 0;
    confirmed[pi] = 0;
  }
  int region = 0;  // 0 = A, 1 = B, 2 = C
  const int64_t total = T.c_end;
  for (int64_t q = blockIdx.x; q < total; q += gridDim.x) {
    const int r = q < T.b_begin ? 0 : (q < T.c_begin ? 1 : 2);
    while (region < r) {  // leaving a region: publish this CTA's tile counts for it
      __syncthreads();
      if (threadIdx.x == 0) publish(T, region, cnt);
#pragma unroll
      for (int pi = 0; pi < kMaxXParts; ++pi) cnt[pi] = 0;
      ++region;
    }
    // locate (part, tile) in the region
    const int64_t base = r == 0 ? 0 : (r == 1 ? T.b_begin : T.c_begin);
    int64_t t = q - base;
    int pi = 0;
    for (; pi < T.nparts; ++pi) {
      const int64_t n = r == 1 ? T.part[pi].tb : T.part[pi].ta;
      if (t < n) break;
      t -= n;
    }
    const XPart& p = T.part[pi];
    Geo<U> geo{p.n4, p.S4, p.rem, p.kp};
    if (r == 0) {
      int o;
      int64_t tt;
      other_slice_tile(p, geo, t, &o, &tt);
      tile_A<M, U>(p, geo, o, tt);
    } else if (r == 1) {
      if (threadIdx.x == 0)
        for (int d = 0; d < p.kp; ++d)
          if (d != p.me && !((confirmed[pi] >> d) & 1)) {
            wait_peer(T, p, d, kPhaseA);
            confirmed[pi] |= 1u << d;
          }
      __syncthreads();
      tile_B<M, U>(p, geo, t);
    } else {
      int o;
      int64_t tt;
      other_slice_tile(p, geo, t, &o, &tt);
      if (threadIdx.x == 0 && !((confirmed[pi] >> (8 + o)) & 1)) {
        wait_peer(T, p, o, kPhaseB);
        confirmed[pi] |= 1u << (8 + o);
      }
      __syncthreads();
      tile_C<M, U>(p, geo, o, tt);
    }
    cnt[pi] += 1;
  }
  // publish the remaining regions (a CTA may end inside A or B)
  while (region < 3) {
    __syncthreads();
    if (threadIdx.x == 0) publish(T, region, cnt);
#pragma unroll
    for (int pi = 0; pi < kMaxXParts; ++pi) cnt[pi] = 0;
    ++region;
  }
  // end of the group: wait until every peer has finished reading my memory
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int pi = 0; pi < T.nparts; ++pi)
      for (int d = 0; d < T.part[pi].kp; ++d)
        if (d != T.part[pi].me) wait_peer(T, T.part[pi], d, kPhaseC);
}

int g_sms = 0;

template <int M, int U>
int launch_m(XTask& T, cudaStream_t stream, std::string* err) {
  static int occ = 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, xgpu_kernel<M, U>, kXThreads, 0) != cudaSuccess || occ < 1)
      occ = 1;
  }
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  // tile geometry per part
  int64_t a = 0, b = 0;
  const int64_t tile = static_cast<int64_t>(kXThreads) * U;
  for (int pi = 0; pi < T.nparts; ++pi) {
    XPart& p = T.part[pi];
    p.n4 = T.n / 4;
    p.rem = static_cast<int32_t>(T.n - 4 * p.n4);
    p.S4 = ((p.n4 + p.kp - 1) / p.kp + tile - 1) / tile * tile;
    int64_t ta = 0, tb = 0;
    for (int o = 0; o < p.kp; ++o) {
      const int64_t lo = std::min(o * p.S4, p.n4), hi = std::min((o + 1) * p.S4, p.n4);
      int64_t t = (hi - lo + tile - 1) / tile;
      if (o == p.kp - 1 && p.rem > 0 && (hi - lo) % tile == 0) ++t;
      if (o == p.me)
        tb = t;
      else
        ta += t;
    }
    p.ta = ta;
    p.tb = tb;
    a += ta;
    b += tb;
  }
  T.b_begin = a;
  T.c_begin = a + b;
  T.c_end = a + b + a;
  const int64_t cap = static_cast<int64_t>(g_sms) * occ;  // all CTAs co-resident
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min(cap, T.c_end)));
  xgpu_kernel<M, U><<<blocks, kXThreads, 0, stream>>>(T);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("xgpu kernel launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

}  // namespace

int launch_xgpu(XTask& T, void* stream, std::string* err) {
  if (T.nparts < 1 || T.nparts > kMaxXParts) {
    *err = "xgpu: bad part count";
    return RP_EINVAL;
  }
  int mmax = 0;
  for (int pi = 0; pi < T.nparts; ++pi) {
    const XPart& p = T.part[pi];
    if (p.m < 1 || p.m > kMaxXLocal || p.kp < 2 || p.kp > kMaxXGpus || p.me < 0 || p.me >= p.kp) {
      *err = "xgpu: bad part descriptor";
      return RP_EINVAL;
    }
    for (int d = 0; d < p.kp; ++d)
      if (!p.src[d] || !p.pflags[d] || (reinterpret_cast<uintptr_t>(p.src[d]) & 15)) {
        *err = "xgpu: peer pointers missing (call rp_peer_import) or misaligned";
        return RP_EINVAL;
      }
    mmax = std::max(mmax, p.m);
  }
  // every cross part of a step must be in ONE launch (two launches on one stream
  // could wait on each other across GPUs), so M is the largest local count
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mmax <= 1) return launch_m<1, 2>(T, s, err);
  if (mmax <= 2) return launch_m<2, 2>(T, s, err);
  if (mmax <= 4) return launch_m<4, 1>(T, s, err);
  return launch_m<8, 1>(T, s, err);
}

}  // namespace rp
