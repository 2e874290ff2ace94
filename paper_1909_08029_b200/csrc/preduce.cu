// Fused SGD + P-Reduce kernel for groups whose members share one GPU.
//
// alg1, steps 2 and 4 in one pass over HBM:
//   y_m    = x_m[j] - lr_m * g_m[j]            for m in G          (step 2)
//   xbar   = (1/|G|) * sum_m y_m                                     (step 4)
//   x_m[j] = xbar                              for m in G
// y is never stored. Non-members are not touched (F^G_uu = 1).
// One launch executes several disjoint groups at once ("non-conflicting
// F^G's can be executed concurrently"): the element range of every
// group is cut into tiles and the persistent grid walks the union of tiles.
//
// Pinned fp32 arithmetic (reading R1): __fmul_rn / __fsub_rn /
// __fadd_rn / __fdiv_rn (no FMA contraction), left fold over members in
// ascending worker id, IEEE division by |G| (never a multiply by fl(1/|G|)).
//
// Memory: per element and member 4 B of x and 4 B of g read, 4 B of x
// written: 12*k bytes per element, the algorithmic minimum (DESIGN.md
// "Roofline"). 128-bit loads/stores; each thread keeps U*2k of them in
// flight; grid = resident CTAs (148 SMs x occupancy).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "rp_internal.h"

namespace rp {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float4 ld_x(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float4 ld_g(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_x(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// y = fl(x - fl(lr*g))
__device__ __forceinline__ float sgd(float x, float g, float lr) { return __fsub_rn(x, __fmul_rn(lr, g)); }

template <int K>
__device__ __forceinline__ float fold_mean(const float (&y)[K]) {
  float s = y[0];
#pragma unroll
  for (int m = 1; m < K; ++m) s = __fadd_rn(s, y[m]);
  return K == 1 ? s : __fdiv_rn(s, static_cast<float>(K));
}

// One tile of group gi: float4 indices [i0, i0 + kThreads*U) of every member.
template <int K, int U>
__device__ __forceinline__ void group_tile(const MultiTask& t, int gi, int64_t i0, int64_t n4) {
  float* x[K];
  const float* g[K];
  float lr[K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    x[m] = t.x[gi * K + m];
    g[m] = t.g[gi * K + m];
    lr[m] = t.lr[gi * K + m];
  }
  float4 xv[U][K], gv[U][K];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + static_cast<int64_t>(u) * kThreads + threadIdx.x;
    if (i < n4) {
#pragma unroll
      for (int m = 0; m < K; ++m) {
        xv[u][m] = ld_x(x[m] + 4 * i);
        if (g[m] != nullptr) gv[u][m] = ld_g(g[m] + 4 * i);
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
        if (g[m] != nullptr) {
          yx[m] = sgd(xv[u][m].x, gv[u][m].x, lr[m]);
          yy[m] = sgd(xv[u][m].y, gv[u][m].y, lr[m]);
          yz[m] = sgd(xv[u][m].z, gv[u][m].z, lr[m]);
          yw[m] = sgd(xv[u][m].w, gv[u][m].w, lr[m]);
        } else {
          yx[m] = xv[u][m].x;
          yy[m] = xv[u][m].y;
          yz[m] = xv[u][m].z;
          yw[m] = xv[u][m].w;
        }
      }
      const float4 r = make_float4(fold_mean<K>(yx), fold_mean<K>(yy), fold_mean<K>(yz), fold_mean<K>(yw));
#pragma unroll
      for (int m = 0; m < K; ++m) st_x(x[m] + 4 * i, r);
    }
  }
}

// Element j of group gi, scalar (the n mod 4 ragged tail).
template <int K>
__device__ __forceinline__ void group_scalar(const MultiTask& t, int gi, int64_t j) {
  float y[K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    const float* g = t.g[gi * K + m];
    const float xj = t.x[gi * K + m][j];
    y[m] = g != nullptr ? sgd(xj, g[j], t.lr[gi * K + m]) : xj;
  }
  const float r = fold_mean<K>(y);
#pragma unroll
  for (int m = 0; m < K; ++m) t.x[gi * K + m][j] = r;
}

// All t.ngroups groups have exactly K members (the engine splits a batch by
// group size, so each instantiation keeps the register budget of its K).
// Persistent grid over ngroups * tiles tiles, groups interleaved tile by tile.
template <int K, int U>
__global__ void __launch_bounds__(kThreads) preduce_multi_kernel(const MultiTask t, const int64_t n4,
                                                                const int64_t n, const int64_t tiles) {
  const int64_t total = tiles * t.ngroups;
  for (int64_t q = blockIdx.x; q < total; q += gridDim.x) {
    const int gi = static_cast<int>(q % t.ngroups);
    group_tile<K, U>(t, gi, (q / t.ngroups) * kThreads * U, n4);
  }
  const int64_t rem = n - 4 * n4;
  if (blockIdx.x == 0 && threadIdx.x < rem * t.ngroups)
    group_scalar<K>(t, static_cast<int>(threadIdx.x / rem), 4 * n4 + threadIdx.x % rem);
}

int g_num_sms = 0;

template <int K, int U>
int launch_k(const MultiTask& t, int64_t n, cudaStream_t stream, std::string* err) {
  static int occ = 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, preduce_multi_kernel<K, U>, kThreads, 0) !=
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
  const int64_t tiles = (n4 + kThreads * U - 1) / (kThreads * U);
  const int64_t want = std::max<int64_t>(1, tiles * t.ngroups);
  const int64_t cap = static_cast<int64_t>(g_num_sms) * occ;
  const int blocks = static_cast<int>(std::min(want, cap));
  preduce_multi_kernel<K, U><<<blocks, kThreads, 0, stream>>>(t, n4, n, tiles);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("preduce kernel launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

}  // namespace

int launch_preduce_multi(const MultiTask& t, int64_t n, void* stream, std::string* err) {
  if (t.ngroups < 1 || t.ngroups > kMaxTasks) {
    *err = "preduce: bad group count";
    return RP_EINVAL;
  }
  const int k = t.group_k[0];
  if (k < 1 || k > RP_MAX_GROUP || k * t.ngroups > kMaxTaskMembers) {
    *err = "preduce: bad group size";
    return RP_EINVAL;
  }
  for (int gi = 0; gi < t.ngroups; ++gi) {
    if (t.group_k[gi] != k || t.group_first[gi] != gi * k) {
      *err = "preduce: groups of one launch must have equal size and packed members";
      return RP_EINVAL;
    }
  }
  for (int i = 0; i < k * t.ngroups; ++i) {
    if (!t.x[i] || (reinterpret_cast<uintptr_t>(t.x[i]) & 15) || (reinterpret_cast<uintptr_t>(t.g[i]) & 15)) {
      *err = "preduce: replica and gradient pointers must be non-null and 16-byte aligned";
      return RP_EINVAL;
    }
  }
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (k) {
    case 1: return launch_k<1, 4>(t, n, s, err);
    case 2: return launch_k<2, 2>(t, n, s, err);
    case 3: return launch_k<3, 2>(t, n, s, err);
    case 4: return launch_k<4, 2>(t, n, s, err);
    case 5: return launch_k<5, 1>(t, n, s, err);
    case 6: return launch_k<6, 1>(t, n, s, err);
    case 7: return launch_k<7, 1>(t, n, s, err);
    case 8: return launch_k<8, 1>(t, n, s, err);
    case 9: return launch_k<9, 1>(t, n, s, err);
    case 10: return launch_k<10, 1>(t, n, s, err);
    case 11: return launch_k<11, 1>(t, n, s, err);
    case 12: return launch_k<12, 1>(t, n, s, err);
    case 13: return launch_k<13, 1>(t, n, s, err);
    case 14: return launch_k<14, 1>(t, n, s, err);
    case 15: return launch_k<15, 1>(t, n, s, err);
    default: return launch_k<16, 1>(t, n, s, err);
  }
}

}  // namespace rp
