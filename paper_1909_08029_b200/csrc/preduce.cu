// Fused SGD + P-Reduce kernel for groups whose members share one GPU.
//
// alg1, steps 2 and 4 in one pass over HBM:
//   y_m    = x_m[j] - lr_m * g_m[j]            for m in G          (step 2)
//   xbar   = (1/|G|) * sum_m y_m                                     (step 4)
//   x_m[j] = xbar                              for m in G
// y is never stored. Non-members are not touched (F^G_uu = 1).
// One launch executes several disjoint groups at once ("non-conflicting
// F^G's can be executed concurrently"): the resident grid is shared
// out among the groups in proportion to their bytes.
//
// Pinned fp32 arithmetic (reading R1): __fmul_rn / __fsub_rn /
// __fadd_rn / __fdiv_rn (no FMA contraction), left fold over members in
// ascending worker id, IEEE division by |G| (never a multiply by fl(1/|G|)).
//
// Memory: per element and member 4 B of x and 4 B of g read, 4 B of x
// written: 12*k bytes per element, the algorithmic minimum (DESIGN.md
// "Roofline"). 128-bit loads/stores with the streaming (.cs, evict-first)
// cache policy: nothing is reused within a step, and the working set of a
// step (2.45 GB at configs[1]) is 20x the L2. Each thread keeps U*2k loads in
// flight; grid = resident CTAs (148 SMs x occupancy).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "rp_internal.h"
#include "update.cuh"

namespace rp {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float4 ld_x(const float* p) {
  float4 v;
  asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float4 ld_g(const float* p) {
  float4 v;
  asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_x(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

template <int K>
__device__ __forceinline__ float fold_mean(const float (&y)[K]) {
  float s = y[0];
#pragma unroll
  for (int m = 1; m < K; ++m) s = __fadd_rn(s, y[m]);
  return K == 1 ? s : __fdiv_rn(s, static_cast<float>(K));
}

__device__ __forceinline__ float4 ld_v(const float* p) {
  float4 v;
  asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

// One tile of the group whose members start at `first`: float4 indices [i0, i0 + kThreads*U)
// of every member. MOM: some member carries a momentum buffer (read and written here).
template <int K, int U, bool MOM>
__device__ __forceinline__ void group_tile(const MultiTask& t, int first, int64_t i0, int64_t n4) {
  float* x[K];
  MemberUpdate up[K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    x[m] = t.x[first + m];
    up[m] = t.u[first + m];
  }
  float4 xv[U][K], gv[U][K], vv[U][MOM ? K : 1];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + static_cast<int64_t>(u) * kThreads + threadIdx.x;
    if (i < n4) {
#pragma unroll
      for (int m = 0; m < K; ++m) {
        xv[u][m] = ld_x(x[m] + 4 * i);
        if (up[m].g != nullptr) gv[u][m] = ld_g(up[m].g + 4 * i);
        if constexpr (MOM)
          if (up[m].v != nullptr) vv[u][m] = ld_v(up[m].v + 4 * i);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + static_cast<int64_t>(u) * kThreads + threadIdx.x;
    if (i < n4) {
      float yx[K], yy[K], yz[K], yw[K];
#pragma unroll
      for (int m = 0; m < K; ++m) {
        float4 vm = MOM ? vv[u][MOM ? m : 0] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 y = step4<MOM>(xv[u][m], gv[u][m], vm, up[m]);
        if constexpr (MOM)
          if (up[m].v != nullptr && up[m].g != nullptr) st_x(up[m].v + 4 * i, vm);
        yx[m] = y.x;
        yy[m] = y.y;
        yz[m] = y.z;
        yw[m] = y.w;
      }
      const float4 r = make_float4(fold_mean<K>(yx), fold_mean<K>(yy), fold_mean<K>(yz), fold_mean<K>(yw));
#pragma unroll
      for (int m = 0; m < K; ++m) st_x(x[m] + 4 * i, r);
    }
  }
}

// Element j of the group whose members start at `first`, scalar (the n mod 4 tail).
template <int K, bool MOM>
__device__ __forceinline__ void group_scalar(const MultiTask& t, int first, int64_t j) {
  float y[K];
#pragma unroll
  for (int m = 0; m < K; ++m) y[m] = step1<MOM>(t.x[first + m][j], t.u[first + m], j);
  const float r = fold_mean<K>(y);
#pragma unroll
  for (int m = 0; m < K; ++m) t.x[first + m][j] = r;
}

// CTA blocks [cta_begin[gi], cta_begin[gi+1]) work on group gi only (CTAs are
// shared out in proportion to each group's bytes), so a CTA runs a single
// K-specialized loop for its whole life. Each CTA grid-strides over its group's
// tiles.
template <int K, int U, bool MOM>
__device__ __forceinline__ void group_loop(const MultiTask& t, int gi, int first, int64_t n4, int64_t n) {
  const int64_t nb = t.cta_begin[gi + 1] - t.cta_begin[gi];
  const int64_t b = static_cast<int64_t>(blockIdx.x) - t.cta_begin[gi];
  const int64_t tiles = (n4 + kThreads * U - 1) / (kThreads * U);
  for (int64_t tile = b; tile < tiles; tile += nb) group_tile<K, U, MOM>(t, first, tile * kThreads * U, n4);
  const int64_t rem = n - 4 * n4;  // ragged tail: first CTA of the group, scalar
  if (b == 0 && threadIdx.x < rem) group_scalar<K, MOM>(t, first, 4 * n4 + threadIdx.x);
}

template <int K, int U, int KMAX, bool MOM>
__device__ __forceinline__ void loop_if(const MultiTask& t, int gi, int first, int64_t n4, int64_t n) {
  if constexpr (K <= KMAX) group_loop<K, U, MOM>(t, gi, first, n4, n);
}

// KMAX bounds the instantiated group sizes (and so the register budget); MINB is the
// resident-CTA floor given to ptxas (RP_PREDUCE_MINB selects 2 for k <= 4, 3 or 4 for
// k <= 8: more warps in flight vs all 2k loads of a thread in registers;
// profiles/r01_hbm_probe_k8.txt).
template <int KMAX, int U, int MINB, bool MOM>
__global__ void __launch_bounds__(kThreads, MINB) preduce_multi_kernel(const MultiTask t, const int64_t n4,
                                                                      const int64_t n) {
  int gi = 0;
  while (gi + 1 < t.ngroups && static_cast<int>(blockIdx.x) >= t.cta_begin[gi + 1]) ++gi;
  const int first = t.group_first[gi];
  switch (t.group_k[gi]) {
    case 1: loop_if<1, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 2: loop_if<2, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 3: loop_if<3, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 4: loop_if<4, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 5: loop_if<5, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 6: loop_if<6, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 7: loop_if<7, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 8: loop_if<8, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 9: loop_if<9, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 10: loop_if<10, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 11: loop_if<11, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 12: loop_if<12, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 13: loop_if<13, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 14: loop_if<14, U, KMAX, MOM>(t, gi, first, n4, n); break;
    case 15: loop_if<15, U, KMAX, MOM>(t, gi, first, n4, n); break;
    default: loop_if<16, U, KMAX, MOM>(t, gi, first, n4, n); break;
  }
}

int g_num_sms = 0;

template <int KMAX, int U, int MINB, bool MOM>
int launch_kmax(MultiTask t, int64_t n, cudaStream_t stream, std::string* err) {
  static int occ = 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, preduce_multi_kernel<KMAX, U, MINB, MOM>, kThreads, 0) !=
            cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  const int64_t n4 = n / 4;
  const int64_t tiles = std::max<int64_t>(1, (n4 + kThreads * U - 1) / (kThreads * U));
  // CTAs in proportion to each group's bytes (k members), at least one, at most its tile count
  int64_t kt = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) kt += t.group_k[gi];
  const int64_t cap = std::max<int64_t>(static_cast<int64_t>(g_num_sms) * occ, t.ngroups);
  int32_t acc = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) {
    t.cta_begin[gi] = acc;
    int64_t share = (cap * t.group_k[gi]) / kt;
    share = std::max<int64_t>(1, std::min(share, tiles));
    acc += static_cast<int32_t>(share);
  }
  t.cta_begin[t.ngroups] = acc;
  preduce_multi_kernel<KMAX, U, MINB, MOM><<<acc, kThreads, 0, stream>>>(t, n4, n);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("preduce kernel launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

}  // namespace

void preload_preduce() {  // every instantiation launch_preduce_multi can pick (see preload_xgpu_ws)
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, preduce_multi_kernel<2, 2, 1, true>);
  cudaFuncGetAttributes(&a, preduce_multi_kernel<4, 1, 1, true>);
  cudaFuncGetAttributes(&a, preduce_multi_kernel<8, 1, 1, true>);
  cudaFuncGetAttributes(&a, preduce_multi_kernel<16, 1, 1, true>);
  cudaFuncGetAttributes(&a, preduce_multi_kernel<2, 2, 1, false>);
  cudaFuncGetAttributes(&a, preduce_multi_kernel<4, 2, 1, false>);
  cudaFuncGetAttributes(&a, preduce_multi_kernel<8, 1, 1, false>);
  cudaFuncGetAttributes(&a, preduce_multi_kernel<16, 1, 1, false>);
}

int launch_preduce_multi(const MultiTask& t, int64_t n, void* stream, std::string* err) {
  if (t.ngroups < 1 || t.ngroups > kMaxTasks) {
    *err = "preduce: bad group count";
    return RP_EINVAL;
  }
  int kmax = 0, nm = 0;
  for (int gi = 0; gi < t.ngroups; ++gi) {
    const int k = t.group_k[gi];
    if (k < 1 || k > RP_MAX_GROUP || t.group_first[gi] != nm || nm + k > kMaxTaskMembers) {
      *err = "preduce: bad group descriptor";
      return RP_EINVAL;
    }
    nm += k;
    kmax = std::max(kmax, k);
  }
  for (int i = 0; i < nm; ++i) {
    if (!t.x[i] || (reinterpret_cast<uintptr_t>(t.x[i]) & 15) || (reinterpret_cast<uintptr_t>(t.u[i].g) & 15) ||
        (reinterpret_cast<uintptr_t>(t.u[i].v) & 15)) {
      *err = "preduce: replica and gradient pointers must be non-null and 16-byte aligned";
      return RP_EINVAL;
    }
  }
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  static int minb = -1;  // RP_PREDUCE_MINB: resident-CTA floor for the k <= 4 and k <= 8 kernels
  if (minb < 0) {
    const char* v = std::getenv("RP_PREDUCE_MINB");
    minb = v && *v ? std::atoi(v) : 0;
  }
  // TMA bulk-copy pipeline (preduce_tma.cu) by default: the warp-specialized kernel with
  // dynamic tile scheduling (variant 7) won the sweeps (+11 % over the static split of
  // variant 5, profiles/r01_split/sweep_*.txt); 5/6 are the statically split warp-specialized
  // variants, 1-4 the CTA-synchronous ones; RP_PREDUCE_TMA=0 selects this file's LDG/STG kernel.
  static int use_tma = -1;
  if (use_tma < 0) {
    const char* v = std::getenv("RP_PREDUCE_TMA");
    use_tma = v && *v ? std::atoi(v) : 7;
  }
  if (use_tma > 0) {
    const int rc = launch_preduce_tma(t, n, stream, err, use_tma);
    if (rc != RP_EINVAL) return rc;
  }
  bool mom = false;
  for (int i = 0; i < nm; ++i) mom = mom || (t.u[i].v != nullptr && t.u[i].g != nullptr);
  if (mom) {  // momentum buffers: a separate instantiation keeps the plain path's registers
    if (kmax <= 2) return launch_kmax<2, 2, 1, true>(t, n, s, err);
    if (kmax <= 4) return launch_kmax<4, 1, 1, true>(t, n, s, err);
    if (kmax <= 8) return launch_kmax<8, 1, 1, true>(t, n, s, err);
    return launch_kmax<16, 1, 1, true>(t, n, s, err);
  }
  if (kmax <= 2) return launch_kmax<2, 2, 1, false>(t, n, s, err);
  if (kmax <= 4)
    return minb == 2 ? launch_kmax<4, 2, 2, false>(t, n, s, err) : launch_kmax<4, 2, 1, false>(t, n, s, err);
  if (kmax <= 8) {
    if (minb == 3) return launch_kmax<8, 1, 3, false>(t, n, s, err);
    if (minb == 4) return launch_kmax<8, 1, 4, false>(t, n, s, err);
    return launch_kmax<8, 1, 1, false>(t, n, s, err);
  }
  return launch_kmax<16, 1, 1, false>(t, n, s, err);
}

}  // namespace rp
