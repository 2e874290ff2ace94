// Intra-GPU fused SGD + P-Reduce with the Tensor Memory Accelerator (TMA) moving the data:
// the same arithmetic as preduce.cu (alg1 steps 2 + 4, pinned fp32
// order of reading R1), but every member's x and g tile is brought into shared memory by
// one cp.async.bulk (completion on an mbarrier, S-stage pipeline), and the mean tile is
// written ONCE to shared memory and pushed to all k member replicas by k bulk stores.
// C persistent CTAs per SM; CTAs are shared out among the launch's groups by bytes.
// Default path for plain SGD steps: the warp-specialized kernel with dynamic tile scheduling
// (variant 7, fp32 and bf16; one producer warp, eight consumer warps, full/empty mbarriers,
// no CTA-wide barrier in the loop, tiles of all groups drawn from one global counter);
// variants 5/6 split the tiles statically; groups of 9-16 members take the CTA-synchronous
// kernel; momentum steps take the LDG kernel of preduce.cu. bf16 replicas (reading R26) use the same bulk
// copies (16 bytes = 8 elements) with fp32 arithmetic and one rounding of the mean.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>

#include "rp_internal.h"
#include "update.cuh"

namespace rp {

namespace {

constexpr int kTThreads = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Shared memory of one CTA: S stages of 2*KMAX tiles (x and g per member), two mean tiles, S barriers.
template <int KMAX, int T, int S>
__host__ __device__ constexpr size_t smem_bytes() {
  return (static_cast<size_t>(S) * 2 * KMAX + 2) * T * sizeof(float4) + S * sizeof(uint64_t);
}

// The CTAs [cta_begin[gi], cta_begin[gi+1]) own group gi; each takes tiles b, b+nb, ...
// fl(s / K) (reading R1). For K = 2^j the product s * 2^-j is exact-scaled and correctly
// rounded exactly like the quotient (both are RNE of the same real number), so it is the
// same bits at a fraction of the cost of the IEEE division sequence.
template <int K>
__device__ __forceinline__ float div_k(float s) {
  if constexpr ((K & (K - 1)) == 0) return __fmul_rn(s, 1.0f / static_cast<float>(K));
  else return __fdiv_rn(s, static_cast<float>(K));
}

// bf16 helpers (reading R26): widening is exact; narrowing is IEEE round-to-nearest-even
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t bf_pack(float lo, float hi) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(lo))) |
         (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(hi))) << 16);
}

// 16 bytes of bf16 (8 elements) of every member -> the rounded mean, packed
template <int K>
__device__ __forceinline__ uint4 mean8_bf16(const float4* stage, int s2k, int T, int e, const MemberUpdate (&up)[K]) {
  float acc[8];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    const uint4 xw = reinterpret_cast<const uint4*>(stage)[(s2k + 2 * m) * T + e];
    const uint32_t xs[4] = {xw.x, xw.y, xw.z, xw.w};
    uint32_t gs[4] = {0, 0, 0, 0};
    if (up[m].g) {
      const uint4 gw = reinterpret_cast<const uint4*>(stage)[(s2k + 2 * m + 1) * T + e];
      gs[0] = gw.x; gs[1] = gw.y; gs[2] = gw.z; gs[3] = gw.w;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float y0 = bf_lo(xs[q]), y1 = bf_hi(xs[q]);
      if (up[m].g) {
        y0 = step_sgd(y0, bf_lo(gs[q]), up[m].lr);
        y1 = step_sgd(y1, bf_hi(gs[q]), up[m].lr);
      }
      acc[2 * q] = m == 0 ? y0 : __fadd_rn(acc[2 * q], y0);
      acc[2 * q + 1] = m == 0 ? y1 : __fadd_rn(acc[2 * q + 1], y1);
    }
  }
  if (K > 1) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = div_k<K>(acc[j]);
  }
  return make_uint4(bf_pack(acc[0], acc[1]), bf_pack(acc[2], acc[3]), bf_pack(acc[4], acc[5]),
                    bf_pack(acc[6], acc[7]));
}

// 16 bytes of fp32 (4 elements) of every member -> the mean
template <int K>
__device__ __forceinline__ float4 mean4_f32(const float4* stage, int s2k, int T, int e, const MemberUpdate (&up)[K]) {
  float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f);
  float sx = 0.f, sy = 0.f, sz = 0.f, sw = 0.f;
#pragma unroll
  for (int m = 0; m < K; ++m) {
    const float4 xv = stage[(s2k + 2 * m) * T + e];
    const float4 gv = up[m].g ? stage[(s2k + 2 * m + 1) * T + e] : xv;
    const float4 y = step4<false>(xv, gv, v0, up[m]);
    sx = m == 0 ? y.x : __fadd_rn(sx, y.x);
    sy = m == 0 ? y.y : __fadd_rn(sy, y.y);
    sz = m == 0 ? y.z : __fadd_rn(sz, y.z);
    sw = m == 0 ? y.w : __fadd_rn(sw, y.w);
  }
  if (K > 1) {
    sx = div_k<K>(sx);
    sy = div_k<K>(sy);
    sz = div_k<K>(sz);
    sw = div_k<K>(sw);
  }
  return make_float4(sx, sy, sz, sw);
}

// ragged tail element j (n mod 4, or n mod 8 for bf16), scalar, same order
template <int K, bool BF>
__device__ __forceinline__ void tail_elem(float* const (&x)[K], const MemberUpdate (&up)[K], int64_t j) {
  float acc = 0.f;
#pragma unroll
  for (int m = 0; m < K; ++m) {
    float y;
    if constexpr (BF) {
      y = __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(x[m])[j]) << 16);
      if (up[m].g)
        y = step_sgd(y, __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(up[m].g)[j]) << 16),
                     up[m].lr);
    } else {
      y = step1<false>(x[m][j], up[m], j);
    }
    acc = m == 0 ? y : __fadd_rn(acc, y);
  }
  if (K > 1) acc = div_k<K>(acc);
#pragma unroll
  for (int m = 0; m < K; ++m) {
    if constexpr (BF) reinterpret_cast<uint16_t*>(x[m])[j] = __bfloat16_as_ushort(__float2bfloat16_rn(acc));
    else x[m][j] = acc;
  }
}

// ---- warp-specialized variant ------------------------------------------------------------
// Warp 8 produces (one elected lane issues the 2K bulk loads of a tile into a free stage),
// warps 0-7 consume: each owns T/8 float4 of every tile, computes its slice of the mean into
// its own double-buffered output slice and bulk-stores it to the k members itself. Stages
// are handed back through an `empty` mbarrier (8 arrivals); there is no CTA-wide barrier in
// the loop, so a warp never waits for the slowest warp of its CTA.
constexpr int kWsConsumers = 8;
constexpr int kWsThreads = 32 * (kWsConsumers + 1);

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int K, int T, int kStages, bool BF>
__device__ void group_ws(const MultiTask& t, int gi, int first, int64_t n4, int64_t n, float4* smem) {
  static_assert(T % (32 * kWsConsumers) == 0, "each consumer lane owns whole float4 columns");
  constexpr int kPerWarp = T / kWsConsumers;
  const int64_t nb = t.cta_begin[gi + 1] - t.cta_begin[gi];
  const int64_t b = static_cast<int64_t>(blockIdx.x) - t.cta_begin[gi];
  const int64_t tiles = (n4 + T - 1) / T;
  const int64_t ntl = tiles > b ? (tiles - b + nb - 1) / nb : 0;
  float4* stage = smem;                         // [kStages][2K][T]
  float4* out = stage + kStages * 2 * K * T;    // [2][T]
  uint64_t* full = reinterpret_cast<uint64_t*>(out + 2 * T);
  uint64_t* empty = full + kStages;
  MemberUpdate up[K];
  float* x[K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    x[m] = t.x[first + m];
    up[m] = t.u[first + m];
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWsConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kWsConsumers) {  // producer
    if (lane == 0) {
      for (int64_t it = 0; it < ntl; ++it) {
        const int s = static_cast<int>(it % kStages);
        if (it >= kStages) mbar_wait(&empty[s], static_cast<uint32_t>((it / kStages - 1) & 1));
        const int64_t base = (b + it * nb) * T;
        const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(T), n4 - base) * 16);
        uint32_t total = 0;
#pragma unroll
        for (int m = 0; m < K; ++m) total += up[m].g ? 2 * bytes : bytes;
        mbar_expect_tx(&full[s], total);
#pragma unroll
        for (int m = 0; m < K; ++m) {
          bulk_load(stage + (s * 2 * K + 2 * m) * T, x[m] + 4 * base, bytes, &full[s]);
          if (up[m].g) bulk_load(stage + (s * 2 * K + 2 * m + 1) * T, up[m].g + 4 * base, bytes, &full[s]);
        }
      }
    }
    return;
  }
  const int e0 = warp * kPerWarp;
  for (int64_t it = 0; it < ntl; ++it) {
    const int s = static_cast<int>(it % kStages);
    const int ob = static_cast<int>(it & 1);
    const int64_t base = (b + it * nb) * T;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(T), n4 - base));
    if (lane == 0) bulk_wait_read1();  // this warp's stores of tile it-2 have read out[ob]
    __syncwarp();
    mbar_wait(&full[s], static_cast<uint32_t>((it / kStages) & 1));
#pragma unroll
    for (int j = 0; j < kPerWarp / 32; ++j) {
      const int e = e0 + j * 32 + lane;
      if (e < cnt) {
        if constexpr (BF)
          reinterpret_cast<uint4*>(out)[ob * T + e] = mean8_bf16<K>(stage, s * 2 * K, T, e, up);
        else
          out[ob * T + e] = mean4_f32<K>(stage, s * 2 * K, T, e, up);
      }
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty[s]);  // stage s read by this warp
      const int mine = max(0, min(kPerWarp, cnt - e0));
      if (mine > 0) {
#pragma unroll
        for (int m = 0; m < K; ++m)
          bulk_store(x[m] + 4 * (base + e0), out + ob * T + e0, static_cast<uint32_t>(mine * 16));
      }
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
  constexpr int kPer = BF ? 8 : 4;
  const int64_t rem = n - kPer * n4;
  if (b == 0 && threadIdx.x < rem) tail_elem<K, BF>(x, up, kPer * n4 + threadIdx.x);
}

// n4 = number of 16-byte vectors per replica (n/4 fp32 or n/8 bf16); n = elements
template <int K, int T, int kStages, bool BF>
__device__ void group_tma(const MultiTask& t, int gi, int first, int64_t n4, int64_t n, float4* smem) {
  const int64_t nb = t.cta_begin[gi + 1] - t.cta_begin[gi];
  const int64_t b = static_cast<int64_t>(blockIdx.x) - t.cta_begin[gi];
  const int64_t tiles = (n4 + T - 1) / T;
  const int64_t ntl = tiles > b ? (tiles - b + nb - 1) / nb : 0;
  float4* stage = smem;                         // [kStages][2K][T]
  float4* out = stage + kStages * 2 * K * T;    // [2][T]
  uint64_t* bar = reinterpret_cast<uint64_t*>(out + 2 * T);
  MemberUpdate up[K];
  float* x[K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    x[m] = t.x[first + m];
    up[m] = t.u[first + m];
  }
  auto issue = [&](int s, int64_t it) {  // thread 0: loads of the CTA's it-th tile into stage s
    const int64_t base = (b + it * nb) * T;
    const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(T), n4 - base) * 16);
    uint32_t total = 0;
#pragma unroll
    for (int m = 0; m < K; ++m) total += up[m].g ? 2 * bytes : bytes;
    mbar_expect_tx(&bar[s], total);
#pragma unroll
    for (int m = 0; m < K; ++m) {
      bulk_load(stage + (s * 2 * K + 2 * m) * T, x[m] + 4 * base, bytes, &bar[s]);
      if (up[m].g) bulk_load(stage + (s * 2 * K + 2 * m + 1) * T, up[m].g + 4 * base, bytes, &bar[s]);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < kStages && s < ntl; ++s) issue(s, s);
  for (int64_t it = 0; it < ntl; ++it) {
    const int s = static_cast<int>(it % kStages);
    const int ob = static_cast<int>(it & 1);
    const int64_t base = (b + it * nb) * T;
    const int64_t cnt = min(static_cast<int64_t>(T), n4 - base);
    if (threadIdx.x == 0) bulk_wait_read1();  // stores of tile it-2 have read out[ob]
    __syncthreads();
    mbar_wait(&bar[s], static_cast<uint32_t>((it / kStages) & 1));
    if constexpr (BF) {
      for (int e = threadIdx.x; e < cnt; e += kTThreads)
        reinterpret_cast<uint4*>(out)[ob * T + e] = mean8_bf16<K>(stage, s * 2 * K, T, e, up);
    } else for (int e = threadIdx.x; e < cnt; e += kTThreads) {
      float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f);
      float yx[K], yy[K], yz[K], yw[K];
#pragma unroll
      for (int m = 0; m < K; ++m) {
        const float4 xv = stage[(s * 2 * K + 2 * m) * T + e];
        const float4 gv = up[m].g ? stage[(s * 2 * K + 2 * m + 1) * T + e] : xv;
        const float4 y = step4<false>(xv, gv, v0, up[m]);
        yx[m] = y.x;
        yy[m] = y.y;
        yz[m] = y.z;
        yw[m] = y.w;
      }
      float sx = yx[0], sy = yy[0], sz = yz[0], sw = yw[0];
#pragma unroll
      for (int m = 1; m < K; ++m) {
        sx = __fadd_rn(sx, yx[m]);
        sy = __fadd_rn(sy, yy[m]);
        sz = __fadd_rn(sz, yz[m]);
        sw = __fadd_rn(sw, yw[m]);
      }
      if (K > 1) {
        const float kf = static_cast<float>(K);
        sx = __fdiv_rn(sx, kf);
        sy = __fdiv_rn(sy, kf);
        sz = __fdiv_rn(sz, kf);
        sw = __fdiv_rn(sw, kf);
      }
      out[ob * T + e] = make_float4(sx, sy, sz, sw);
    }
    fence_async_smem();
    __syncthreads();  // stage s consumed, out[ob] complete
    if (threadIdx.x == 0) {
      if (it + kStages < ntl) issue(s, it + kStages);
#pragma unroll
      for (int m = 0; m < K; ++m) bulk_store(x[m] + 4 * base, out + ob * T, static_cast<uint32_t>(cnt * 16));
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
  // ragged tail (n mod 4, or n mod 8 for bf16): first CTA of the group, scalar, same order
  constexpr int kPer = BF ? 8 : 4;
  const int64_t rem = n - kPer * n4;
  if constexpr (BF) {
    if (b == 0 && threadIdx.x < rem) {
      const int64_t j = kPer * n4 + threadIdx.x;
      float acc = 0.f;
#pragma unroll
      for (int m = 0; m < K; ++m) {
        const uint16_t* xm = reinterpret_cast<const uint16_t*>(x[m]);
        float y = __uint_as_float(static_cast<uint32_t>(xm[j]) << 16);
        if (up[m].g)
          y = step_sgd(y, __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(up[m].g)[j]) << 16),
                       up[m].lr);
        acc = m == 0 ? y : __fadd_rn(acc, y);
      }
      if (K > 1) acc = __fdiv_rn(acc, static_cast<float>(K));
      const uint16_t r = __bfloat16_as_ushort(__float2bfloat16_rn(acc));
#pragma unroll
      for (int m = 0; m < K; ++m) reinterpret_cast<uint16_t*>(x[m])[j] = r;
    }
    return;
  }
  if (b == 0 && threadIdx.x < rem) {
    const int64_t j = 4 * n4 + threadIdx.x;
    float y[K];
#pragma unroll
    for (int m = 0; m < K; ++m) y[m] = step1<false>(x[m][j], up[m], j);
    float s = y[0];
#pragma unroll
    for (int m = 1; m < K; ++m) s = __fadd_rn(s, y[m]);
    if (K > 1) s = __fdiv_rn(s, static_cast<float>(K));
#pragma unroll
    for (int m = 0; m < K; ++m) x[m][j] = s;
  }
}

template <int K, int KMAX, int T, int S, bool BF>
__device__ __forceinline__ void tma_if(const MultiTask& t, int gi, int first, int64_t n4, int64_t n, float4* smem) {
  if constexpr (K <= KMAX) group_tma<K, T, S, BF>(t, gi, first, n4, n, smem);
}

template <int KMAX, int T, int S, int C, bool BF>
__global__ void __launch_bounds__(kTThreads, C) preduce_tma_kernel(const MultiTask t, const int64_t n4,
                                                                   const int64_t n) {
  extern __shared__ __align__(128) float4 tsmem[];
  int gi = 0;
  while (gi + 1 < t.ngroups && static_cast<int>(blockIdx.x) >= t.cta_begin[gi + 1]) ++gi;
  const int first = t.group_first[gi];
  switch (t.group_k[gi]) {
    case 1: tma_if<1, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 2: tma_if<2, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 3: tma_if<3, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 4: tma_if<4, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 5: tma_if<5, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 6: tma_if<6, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 7: tma_if<7, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 8: tma_if<8, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 9: tma_if<9, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 10: tma_if<10, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 11: tma_if<11, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 12: tma_if<12, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 13: tma_if<13, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 14: tma_if<14, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    case 15: tma_if<15, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
    default: tma_if<16, KMAX, T, S, BF>(t, gi, first, n4, n, tsmem); break;
  }
}

template <int K, int KMAX, int T, int S, bool BF>
__device__ __forceinline__ void ws_if(const MultiTask& t, int gi, int first, int64_t n4, int64_t n, float4* smem) {
  if constexpr (K <= KMAX) group_ws<K, T, S, BF>(t, gi, first, n4, n, smem);
}

template <int KMAX, int T, int S, int C, bool BF>
__global__ void __launch_bounds__(kWsThreads, C) preduce_ws_kernel(const MultiTask t, const int64_t n4,
                                                                   const int64_t n) {
  extern __shared__ __align__(128) float4 wsmem[];
  int gi = 0;
  while (gi + 1 < t.ngroups && static_cast<int>(blockIdx.x) >= t.cta_begin[gi + 1]) ++gi;
  const int first = t.group_first[gi];
  switch (t.group_k[gi]) {
    case 1: ws_if<1, KMAX, T, S, BF>(t, gi, first, n4, n, wsmem); break;
    case 2: ws_if<2, KMAX, T, S, BF>(t, gi, first, n4, n, wsmem); break;
    case 3: ws_if<3, KMAX, T, S, BF>(t, gi, first, n4, n, wsmem); break;
    case 4: ws_if<4, KMAX, T, S, BF>(t, gi, first, n4, n, wsmem); break;
    case 5: ws_if<5, KMAX, T, S, BF>(t, gi, first, n4, n, wsmem); break;
    case 6: ws_if<6, KMAX, T, S, BF>(t, gi, first, n4, n, wsmem); break;
    case 7: ws_if<7, KMAX, T, S, BF>(t, gi, first, n4, n, wsmem); break;
    default: ws_if<8, KMAX, T, S, BF>(t, gi, first, n4, n, wsmem); break;
  }
}

// ---- warp-specialized kernel with dynamic tile scheduling (variant 7) --------------------
// Same pipeline and arithmetic as group_ws, but tiles are handed out at run time from one
// global counter over ALL groups of the launch (tile id -> group id % ngroups, tile
// id / ngroups), so any CTA works on any group and a CTA that becomes resident late (another
// kernel held its SM, e.g. the step's cross-GPU launch on a second stream) simply finds
// fewer tiles left: no static split, no tail from unequal CTA start times. The producer
// fetches its next tile id one tile ahead (atomicAdd latency hidden behind the bulk loads)
// and passes it to the consumers in shared memory beside the stage (published by the
// stage's mbarrier arrive, release/acquire at CTA scope). The last CTA to finish resets the
// launch's counter pair, so the next launch that takes this ring slot finds zeros.
constexpr int kDynSlots = 4096;

template <int K, int T, bool BF>
__device__ __forceinline__ void dyn_consume(const MultiTask& t, int g, int64_t base, int cnt, const float4* stage,
                                            int s2, float4* out, int ob, int e0, int lane) {
  constexpr int kPerWarp = T / kWsConsumers;
  MemberUpdate up[K];
  const int first = t.group_first[g];
#pragma unroll
  for (int m = 0; m < K; ++m) up[m] = t.u[first + m];
#pragma unroll
  for (int j = 0; j < kPerWarp / 32; ++j) {
    const int e = e0 + j * 32 + lane;
    if (e < cnt) {
      if constexpr (BF)
        reinterpret_cast<uint4*>(out)[ob * T + e] = mean8_bf16<K>(stage, s2, T, e, up);
      else
        out[ob * T + e] = mean4_f32<K>(stage, s2, T, e, up);
    }
  }
}

template <int K, int KMAX, int T, bool BF>
__device__ __forceinline__ void dyn_consume_if(const MultiTask& t, int g, int64_t base, int cnt, const float4* stage,
                                               int s2, float4* out, int ob, int e0, int lane) {
  if constexpr (K <= KMAX) dyn_consume<K, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane);
}

template <int KMAX, int T, bool BF>
__device__ __forceinline__ void dyn_tail(const MultiTask& t, int g, int64_t j) {
  const int first = t.group_first[g];
  switch (t.group_k[g]) {
#define RP_DYN_TAIL(KK)                                                  \
  case KK:                                                               \
    if constexpr (KK <= KMAX) {                                          \
      float* x[KK];                                                      \
      MemberUpdate up[KK];                                               \
      for (int m = 0; m < KK; ++m) {                                     \
        x[m] = t.x[first + m];                                           \
        up[m] = t.u[first + m];                                          \
      }                                                                  \
      tail_elem<KK, BF>(x, up, j);                                       \
    }                                                                    \
    break;
    RP_DYN_TAIL(1) RP_DYN_TAIL(2) RP_DYN_TAIL(3) RP_DYN_TAIL(4) RP_DYN_TAIL(5) RP_DYN_TAIL(6) RP_DYN_TAIL(7)
    RP_DYN_TAIL(8)
#undef RP_DYN_TAIL
    default: break;
  }
}

template <int KMAX, int T, int S, int C, bool BF>
__global__ void __launch_bounds__(kWsThreads, C) preduce_dyn_kernel(const MultiTask t, const int64_t n4,
                                                                    const int64_t n, int* ctr) {
  static_assert(T % (32 * kWsConsumers) == 0, "each consumer lane owns whole float4 columns");
  constexpr int kPerWarp = T / kWsConsumers;
  extern __shared__ __align__(128) float4 dsmem[];
  float4* stage = dsmem;                        // [S][2 KMAX][T]
  float4* out = stage + S * 2 * KMAX * T;       // [2][T]
  uint64_t* full = reinterpret_cast<uint64_t*>(out + 2 * T);
  uint64_t* empty = full + S;
  volatile int64_t* tile_of = reinterpret_cast<volatile int64_t*>(empty + S);  // [S]
  const int64_t tiles = (n4 + T - 1) / T;
  const int64_t total = tiles * t.ngroups;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWsConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kWsConsumers) {  // producer
    if (lane == 0) {
      // t.tiles_per_cta > 0: the CTA retires after that many tiles, so the block scheduler
      // regularly frees SM slots (a concurrent cross-GPU launch on a higher-priority stream
      // takes them first); 0: persistent until the counter runs out
      // Tile ids are drawn kDynBatch at a time (one atomic per batch: a single-group launch
      // needs ~4e8 tiles/s, more than one L2 address serves), the next batch one batch ahead.
      unsigned long long* const c0 = reinterpret_cast<unsigned long long*>(ctr);
      const int kDynBatch = t.dyn_batch > 0 ? t.dyn_batch : 1;
      const int64_t quota = t.tiles_per_cta > 0
                                ? (static_cast<int64_t>(t.tiles_per_cta) + kDynBatch - 1) / kDynBatch * kDynBatch
                                : INT64_MAX;
      int64_t batch = static_cast<int64_t>(atomicAdd(c0, static_cast<unsigned long long>(kDynBatch)));
      int64_t nextb = 0;
      int j = 0, s = 0;
      uint32_t phase = 0;
      for (int64_t it = 0;; ++it) {  // no divisions on the producer's critical path
        if (it >= S) mbar_wait(&empty[s], phase ^ 1u);
        if (j == kDynBatch) {
          batch = nextb;
          j = 0;
        }
        if (j == 0 && it + kDynBatch < quota)
          nextb = static_cast<int64_t>(atomicAdd(c0, static_cast<unsigned long long>(kDynBatch)));
        const int64_t id = it < quota ? batch + j : total;
        ++j;
        tile_of[s] = id;
        if (id >= total) {
          mbar_arrive(&full[s]);  // end marker: phase completes with no bytes
          break;
        }
        const uint32_t id32 = static_cast<uint32_t>(id);  // total < 2^31 (checked by the launcher)
        const uint32_t ng = static_cast<uint32_t>(t.ngroups);
        const uint32_t tq = id32 / ng;
        const int g = static_cast<int>(id32 - tq * ng);
        const int first = t.group_first[g], K = t.group_k[g];
        const int64_t base = static_cast<int64_t>(tq) * T;
        const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(T), n4 - base) * 16);
        uint32_t tot = 0;
        for (int m = 0; m < K; ++m) tot += t.u[first + m].g ? 2 * bytes : bytes;
        mbar_expect_tx(&full[s], tot);
        for (int m = 0; m < K; ++m) {
          bulk_load(stage + (s * 2 * KMAX + 2 * m) * T, t.x[first + m] + 4 * base, bytes, &full[s]);
          if (t.u[first + m].g)
            bulk_load(stage + (s * 2 * KMAX + 2 * m + 1) * T, t.u[first + m].g + 4 * base, bytes, &full[s]);
        }
        if (++s == S) {
          s = 0;
          phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    const int e0 = warp * kPerWarp;
    for (int64_t it = 0;; ++it) {
      const int s = static_cast<int>(it % S);
      const int ob = static_cast<int>(it & 1);
      if (lane == 0) bulk_wait_read1();  // this warp's stores of tile it-2 have read out[ob]
      __syncwarp();
      mbar_wait(&full[s], static_cast<uint32_t>((it / S) & 1));
      const int64_t id = tile_of[s];
      if (id >= total) break;
      const uint32_t ng = static_cast<uint32_t>(t.ngroups);
      const uint32_t tq = static_cast<uint32_t>(id) / ng;
      const int g = static_cast<int>(static_cast<uint32_t>(id) - tq * ng);
      const int64_t base = static_cast<int64_t>(tq) * T;
      const int cnt = static_cast<int>(min(static_cast<int64_t>(T), n4 - base));
      const int s2 = s * 2 * KMAX;
      const int K = t.group_k[g];
      switch (K) {
        case 1: dyn_consume_if<1, KMAX, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane); break;
        case 2: dyn_consume_if<2, KMAX, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane); break;
        case 3: dyn_consume_if<3, KMAX, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane); break;
        case 4: dyn_consume_if<4, KMAX, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane); break;
        case 5: dyn_consume_if<5, KMAX, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane); break;
        case 6: dyn_consume_if<6, KMAX, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane); break;
        case 7: dyn_consume_if<7, KMAX, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane); break;
        default: dyn_consume_if<8, KMAX, T, BF>(t, g, base, cnt, stage, s2, out, ob, e0, lane); break;
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[s]);  // stage s read by this warp
        const int mine = max(0, min(kPerWarp, cnt - e0));
        if (mine > 0) {
          const int first = t.group_first[g];
          for (int m = 0; m < K; ++m)
            bulk_store(t.x[first + m] + 4 * (base + e0), out + ob * T + e0, static_cast<uint32_t>(mine * 16));
        }
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  // ragged tail (n mod 4, or n mod 8 for bf16) of every group: CTA 0, scalar, same order
  constexpr int kPer = BF ? 8 : 4;
  const int64_t rem = n - kPer * n4;
  if (blockIdx.x == 0 && threadIdx.x < rem)
    for (int g = 0; g < t.ngroups; ++g) dyn_tail<KMAX, T, BF>(t, g, kPer * n4 + threadIdx.x);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(reinterpret_cast<unsigned long long*>(ctr) + 1, 1ull) == gridDim.x - 1) {
      reinterpret_cast<unsigned long long*>(ctr)[0] = 0;  // every CTA has drawn its end marker
      reinterpret_cast<unsigned long long*>(ctr)[1] = 0;
    }
  }
}

int g_sms_tma = 0;

// CTAs of one launch shared out among its groups in proportion to their member counts
void share_ctas(MultiTask& t, int64_t cap) {
  int64_t kt = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) kt += t.group_k[gi];
  int32_t acc = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) {
    t.cta_begin[gi] = acc;
    acc += static_cast<int32_t>(std::max<int64_t>(1, (cap * t.group_k[gi]) / kt));
  }
  t.cta_begin[t.ngroups] = acc;
}

int sms() {
  if (g_sms_tma == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_tma, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms_tma <= 0) g_sms_tma = 148;
  }
  return g_sms_tma;
}

template <int KMAX, int T, int S, int C, bool BF>
int launch_ws(MultiTask t, int64_t n, cudaStream_t stream, std::string* err) {
  constexpr size_t smem = (static_cast<size_t>(S) * 2 * KMAX + 2) * T * sizeof(float4) + 2 * S * sizeof(uint64_t);
  static_assert(smem * C <= 226 * 1024, "C CTAs must fit one SM");
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(preduce_ws_kernel<KMAX, T, S, C, BF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
      *err = "preduce_ws: shared memory attribute";
      return RP_ECUDA;
    }
    attr = true;
  }
  // a concurrent cross-GPU launch holds t.reserve_sms SMs: every CTA of this grid is
  // resident from the start on the others (persistent CTAs, static tile split)
  const int64_t free_sms = std::max<int64_t>(1, sms() - std::max(0, t.reserve_sms));
  share_ctas(t, std::max<int64_t>(free_sms * C, t.ngroups));
  preduce_ws_kernel<KMAX, T, S, C, BF><<<t.cta_begin[t.ngroups], kWsThreads, smem, stream>>>(t, n / (BF ? 8 : 4), n);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("preduce_ws launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

// ring of per-launch counter pairs (next tile, CTAs done), one ring per device
unsigned long long* dyn_counters(std::string* err) {
  static std::mutex mu;
  static unsigned long long* ring[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!ring[dev]) {
    if (cudaMalloc(&ring[dev], kDynSlots * 2 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(ring[dev], 0, kDynSlots * 2 * sizeof(unsigned long long)) != cudaSuccess) {
      *err = "preduce_dyn: counter ring allocation failed";
      ring[dev] = nullptr;
      return nullptr;
    }
  }
  return ring[dev];
}

template <int KMAX, int T, int S, int C, bool BF>
int launch_dyn(MultiTask t, int64_t n, cudaStream_t stream, std::string* err) {
  constexpr size_t smem = (static_cast<size_t>(S) * 2 * KMAX + 2) * T * sizeof(float4) + 2 * S * sizeof(uint64_t) +
                          S * sizeof(int64_t);
  static_assert(smem * C <= 226 * 1024, "C CTAs must fit one SM");
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(preduce_dyn_kernel<KMAX, T, S, C, BF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
      *err = "preduce_dyn: shared memory attribute";
      return RP_ECUDA;
    }
    attr = true;
  }
  // tile ids per atomic (sweep profiles/r01_kernel_choice/batch_sweep.txt, ms/step at N=1):
  // 1: cfg2 0.3616, cfg2ii 0.3785, bf16 0.1934; 2: 0.3639, 0.3640, 0.1905; 4: 0.3669, 0.3661,
  // 0.1926; 8: 0.3715, 0.3708, 0.1966 -> 2 for every launch (RP_DYN_BATCH overrides)
  static int batch_env = -1;  // RP_DYN_BATCH: tile ids per atomic (0 = default 2)
  if (batch_env < 0) {
    const char* v = std::getenv("RP_DYN_BATCH");
    batch_env = v && *v ? std::atoi(v) : 0;
  }
  t.dyn_batch = batch_env > 0 ? batch_env : 2;
  if ((n / (BF ? 8 : 4) + T) / T * t.ngroups >= (int64_t{1} << 31)) {
    *err = "preduce_dyn: more than 2^31 tiles";
    return RP_EINVAL;
  }
  unsigned long long* ring = dyn_counters(err);
  if (!ring) return RP_ECUDA;
  static std::atomic<uint64_t> next_slot{0};
  int* ctr = reinterpret_cast<int*>(ring + 2 * (next_slot.fetch_add(1) % kDynSlots));
  int64_t grid = static_cast<int64_t>(sms()) * C;
  if (t.tiles_per_cta > 0) {  // enough retiring CTAs to cover every tile
    const int64_t per = BF ? 8 : 4;
    const int64_t tiles = ((n / per) + T - 1) / T * t.ngroups;
    grid = std::max<int64_t>(1, (tiles + t.tiles_per_cta - 1) / t.tiles_per_cta);
  }
  preduce_dyn_kernel<KMAX, T, S, C, BF><<<static_cast<unsigned>(grid), kWsThreads, smem, stream>>>(t, n / (BF ? 8 : 4), n,
                                                                                                ctr);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("preduce_dyn launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

template <bool BF>
int launch_dyn_variant(int kmax, MultiTask t, int64_t n, cudaStream_t s, std::string* err) {
  // beside a cross-GPU launch (reserve_sms > 0): one stage less, so two CTAs still fit an
  // SM next to a cross-kernel CTA (80 KB + 80 KB + 32 KB)
  if (t.reserve_sms > 0 && kmax <= 3) return launch_dyn<3, 256, 3, 2, BF>(t, n, s, err);
  if (t.reserve_sms > 0 && kmax <= 4) return launch_dyn<4, 256, 2, 2, BF>(t, n, s, err);
  if (kmax <= 3) return launch_dyn<3, 256, 4, 2, BF>(t, n, s, err);
  if (kmax <= 4) return launch_dyn<4, 256, 3, 2, BF>(t, n, s, err);
  return launch_dyn<8, 256, 3, 1, BF>(t, n, s, err);
}

// warp-specialized variants: 5 = 4 KB tiles (2 CTAs/SM where they fit), 6 = 8 KB tiles
template <bool BF>
int launch_ws_variant(int variant, int kmax, MultiTask t, int64_t n, cudaStream_t s, std::string* err) {
  if (variant == 6) {
    if (kmax <= 3) return launch_ws<3, 512, 3, 1, BF>(t, n, s, err);
    if (kmax <= 4) return launch_ws<4, 512, 2, 1, BF>(t, n, s, err);
    return launch_ws<8, 256, 3, 1, BF>(t, n, s, err);
  }
  if (kmax <= 3) return launch_ws<3, 256, 4, 2, BF>(t, n, s, err);
  if (kmax <= 4) return launch_ws<4, 256, 3, 2, BF>(t, n, s, err);
  static int k8 = -1;  // RP_WS_K8: stages for 5..8 members (sweep)
  if (k8 < 0) {
    const char* v = std::getenv("RP_WS_K8");
    k8 = v && *v ? std::atoi(v) : 3;
  }
  if (k8 == 2) return launch_ws<8, 256, 2, 1, BF>(t, n, s, err);
  return launch_ws<8, 256, 3, 1, BF>(t, n, s, err);
}

template <int KMAX, int T, int S, int C, bool BF = false>
int launch_tma(MultiTask t, int64_t n, cudaStream_t stream, std::string* err) {
  static_assert(C == 1 || smem_bytes<KMAX, T, S>() * C <= 226 * 1024, "C CTAs must fit one SM");
  const size_t smem = smem_bytes<KMAX, T, S>();
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(preduce_tma_kernel<KMAX, T, S, C, BF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
      *err = "preduce_tma: shared memory attribute";
      return RP_ECUDA;
    }
    attr = true;
  }
  if (g_sms_tma == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_tma, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms_tma <= 0) g_sms_tma = 148;
  }
  int64_t kt = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) kt += t.group_k[gi];
  const int64_t cap = std::max<int64_t>(static_cast<int64_t>(g_sms_tma) * C, t.ngroups);  // C CTAs per SM
  int32_t acc = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) {
    t.cta_begin[gi] = acc;
    acc += static_cast<int32_t>(std::max<int64_t>(1, (cap * t.group_k[gi]) / kt));
  }
  t.cta_begin[t.ngroups] = acc;
  preduce_tma_kernel<KMAX, T, S, C, BF><<<acc, kTThreads, smem, stream>>>(t, n / (BF ? 8 : 4), n);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("preduce_tma launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

}  // namespace

// Returns RP_EINVAL (caller falls back to the LDG kernel) for shapes it does not cover.
template <bool BF>
void tma_touch() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, preduce_dyn_kernel<3, 256, 3, 2, BF>);
  cudaFuncGetAttributes(&a, preduce_dyn_kernel<4, 256, 2, 2, BF>);
  cudaFuncGetAttributes(&a, preduce_dyn_kernel<3, 256, 4, 2, BF>);
  cudaFuncGetAttributes(&a, preduce_dyn_kernel<4, 256, 3, 2, BF>);
  cudaFuncGetAttributes(&a, preduce_dyn_kernel<8, 256, 3, 1, BF>);
  cudaFuncGetAttributes(&a, preduce_ws_kernel<3, 256, 4, 2, BF>);
  cudaFuncGetAttributes(&a, preduce_ws_kernel<4, 256, 3, 2, BF>);
  cudaFuncGetAttributes(&a, preduce_ws_kernel<8, 256, 3, 1, BF>);
  cudaFuncGetAttributes(&a, preduce_ws_kernel<8, 256, 2, 1, BF>);
  cudaFuncGetAttributes(&a, preduce_tma_kernel<16, 64, 6, 1, BF>);
}

// every default-path instantiation (variant 7 + its fallbacks; see preload_xgpu_ws)
void preload_preduce_tma() {
  tma_touch<false>();
  tma_touch<true>();
}

int launch_preduce_tma(const MultiTask& t, int64_t n, void* stream, std::string* err, int variant, bool bf16) {
  int kmax = 0;
  int nm = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) {
    kmax = std::max(kmax, t.group_k[gi]);
    nm += t.group_k[gi];
  }
  for (int i = 0; i < nm; ++i)
    if (t.u[i].v != nullptr) return RP_EINVAL;  // momentum: LDG kernel
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  // variant 7 (dynamic tiles) pays off on large launches; below ~1 GB of algorithmic traffic
  // (e.g. one lone SGD worker of ResNet-50 size: 0.0763 vs 0.0518 ms) the statically split
  // kernel is faster, unless a concurrent cross-GPU launch needs the dynamic one
  static int64_t min_bytes = -1;  // RP_DYN_MIN_BYTES (tests set 0 to force variant 7 everywhere)
  if (min_bytes < 0) {
    const char* v = std::getenv("RP_DYN_MIN_BYTES");
    min_bytes = v && *v ? std::atoll(v) : (int64_t{1} << 30);
  }
  const int64_t launch_bytes = static_cast<int64_t>(nm) * n * (bf16 ? 6 : 12);
  if (variant == 7 && t.reserve_sms == 0 && launch_bytes < min_bytes && kmax <= 8)
    return bf16 ? launch_ws_variant<true>(6, kmax, t, n, s, err) : launch_ws_variant<false>(5, kmax, t, n, s, err);
  if ((variant == 7 || t.reserve_sms > 0) && kmax <= 8)
    return bf16 ? launch_dyn_variant<true>(kmax, t, n, s, err) : launch_dyn_variant<false>(kmax, t, n, s, err);
  if ((variant == 5 || variant == 6) && kmax <= 8) {
    return bf16 ? launch_ws_variant<true>(variant, kmax, t, n, s, err)
                : launch_ws_variant<false>(variant, kmax, t, n, s, err);
  }
  if (bf16) {  // bf16 replicas (reading R26): the only intra-GPU kernel for them
    if (kmax <= 3) return launch_tma<3, 256, 4, 2, true>(t, n, s, err);
    if (kmax <= 4) return launch_tma<4, 128, 6, 2, true>(t, n, s, err);
    if (kmax <= 8) return launch_tma<8, 128, 6, 1, true>(t, n, s, err);
    return launch_tma<16, 64, 6, 1, true>(t, n, s, err);
  }
  if (kmax > 16 || n < 4) return RP_EINVAL;
  if (kmax > 8) return launch_tma<16, 64, 6, 1>(t, n, s, err);
  // (KMAX, tile float4s T, stages S, CTAs per SM C) variants for the sweep in scripts/tma_local.sh
  if (kmax <= 4) {
    switch (variant) {
      case 1: return launch_tma<4, 512, 3, 1>(t, n, s, err);
      case 2: return launch_tma<4, 256, 4, 1>(t, n, s, err);
      case 3: return kmax <= 3 ? launch_tma<3, 256, 4, 2>(t, n, s, err) : launch_tma<4, 128, 6, 2>(t, n, s, err);
      case 4: return launch_tma<4, 128, 6, 2>(t, n, s, err);
      default: return kmax <= 3 ? launch_tma<3, 128, 8, 2>(t, n, s, err) : launch_tma<4, 128, 6, 2>(t, n, s, err);
    }
  }
  switch (variant) {
    case 1: return launch_tma<8, 256, 3, 1>(t, n, s, err);
    case 2: return launch_tma<8, 128, 4, 1>(t, n, s, err);
    case 3: return launch_tma<8, 128, 6, 1>(t, n, s, err);
    case 4: return launch_tma<8, 64, 6, 2>(t, n, s, err);
    default: return launch_tma<8, 128, 3, 2>(t, n, s, err);
  }
}

}  // namespace rp
