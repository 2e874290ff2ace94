// Intra-GPU fused SGD + P-Reduce with the Tensor Memory Accelerator (TMA) moving the data:
// the same arithmetic as preduce.cu (alg1 steps 2 + 4, pinned fp32
// order of reading R1), but every member's x and g tile is brought into shared memory by
// one cp.async.bulk (completion on an mbarrier, S-stage pipeline), and the mean tile is
// written ONCE to shared memory and pushed to all k member replicas by k bulk stores.
// C persistent CTAs per SM; CTAs are shared out among the launch's groups by bytes.
// Default path for plain SGD steps (variant 3, see launch_preduce_multi); momentum steps
// and groups larger than 8 take the LDG kernel of preduce.cu.
#include <cuda_runtime.h>

#include <algorithm>
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
template <int K, int T, int kStages>
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
    for (int e = threadIdx.x; e < cnt; e += kTThreads) {
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
  // ragged n mod 4 tail: first CTA of the group, scalar (pinned order as above)
  const int64_t rem = n - 4 * n4;
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

template <int K, int KMAX, int T, int S>
__device__ __forceinline__ void tma_if(const MultiTask& t, int gi, int first, int64_t n4, int64_t n, float4* smem) {
  if constexpr (K <= KMAX) group_tma<K, T, S>(t, gi, first, n4, n, smem);
}

template <int KMAX, int T, int S, int C>
__global__ void __launch_bounds__(kTThreads, C) preduce_tma_kernel(const MultiTask t, const int64_t n4,
                                                                   const int64_t n) {
  extern __shared__ __align__(128) float4 tsmem[];
  int gi = 0;
  while (gi + 1 < t.ngroups && static_cast<int>(blockIdx.x) >= t.cta_begin[gi + 1]) ++gi;
  const int first = t.group_first[gi];
  switch (t.group_k[gi]) {
    case 1: tma_if<1, KMAX, T, S>(t, gi, first, n4, n, tsmem); break;
    case 2: tma_if<2, KMAX, T, S>(t, gi, first, n4, n, tsmem); break;
    case 3: tma_if<3, KMAX, T, S>(t, gi, first, n4, n, tsmem); break;
    case 4: tma_if<4, KMAX, T, S>(t, gi, first, n4, n, tsmem); break;
    case 5: tma_if<5, KMAX, T, S>(t, gi, first, n4, n, tsmem); break;
    case 6: tma_if<6, KMAX, T, S>(t, gi, first, n4, n, tsmem); break;
    case 7: tma_if<7, KMAX, T, S>(t, gi, first, n4, n, tsmem); break;
    default: tma_if<8, KMAX, T, S>(t, gi, first, n4, n, tsmem); break;
  }
}

int g_sms_tma = 0;

template <int KMAX, int T, int S, int C>
int launch_tma(MultiTask t, int64_t n, cudaStream_t stream, std::string* err) {
  static_assert(C == 1 || smem_bytes<KMAX, T, S>() * C <= 226 * 1024, "C CTAs must fit one SM");
  const size_t smem = smem_bytes<KMAX, T, S>();
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(preduce_tma_kernel<KMAX, T, S, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  preduce_tma_kernel<KMAX, T, S, C><<<acc, kTThreads, smem, stream>>>(t, n / 4, n);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("preduce_tma launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

}  // namespace

// Returns RP_EINVAL (caller falls back to the LDG kernel) for shapes it does not cover.
int launch_preduce_tma(const MultiTask& t, int64_t n, void* stream, std::string* err, int variant) {
  int kmax = 0;
  int nm = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) {
    kmax = std::max(kmax, t.group_k[gi]);
    nm += t.group_k[gi];
  }
  for (int i = 0; i < nm; ++i)
    if (t.u[i].v != nullptr) return RP_EINVAL;  // momentum: LDG kernel
  if (kmax > 8 || n < 4) return RP_EINVAL;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
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
