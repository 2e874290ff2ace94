// Harness kernels for the NCCL baselines of bench.py, not the method's path.
//
// The paper's own P-Reduce is "NCCL all-reduce within the group" on a per-group communicator
// (§6); the global All-Reduce baseline is Horovod/NCCL. With several
// simulated workers per GPU a baseline needs a local pre-sum (NCCL allows one rank per GPU) and
// a local broadcast of the mean. These two kernels make that fair: one pass that applies alg1
// step 2 and folds the GPU's members (12 B/element/member read+written at most once), and one
// pass that writes s / k into every member. NCCL sums the per-GPU partials in between.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "rp_internal.h"

namespace rp {
namespace {

constexpr int kBThreads = 256;
constexpr int kBMax = 16;

struct PresumArgs {
  const float* x[kBMax];
  const float* g[kBMax];
  int32_t m;
};
struct ScatterArgs {
  float* x[kBMax];
  int32_t m;
};

int grid_for(int64_t n4) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n4 + kBThreads - 1) / kBThreads, 4LL * sms)));
}

// out = fl(...fl(y_0 + y_1) + ...), y_m = fl(x_m - fl(lr g_m)) (reading R1 order on one GPU)
__global__ void __launch_bounds__(kBThreads) presum_kernel(const PresumArgs a, int64_t n, float lr,
                                                           float* __restrict__ out) {
  const int64_t n4 = n / 4, stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int m = 0; m < a.m; ++m) {
      const float4 x = __ldcs(reinterpret_cast<const float4*>(a.x[m]) + i);
      const float4 g = __ldcs(reinterpret_cast<const float4*>(a.g[m]) + i);
      const float4 y = make_float4(__fsub_rn(x.x, __fmul_rn(lr, g.x)), __fsub_rn(x.y, __fmul_rn(lr, g.y)),
                                   __fsub_rn(x.z, __fmul_rn(lr, g.z)), __fsub_rn(x.w, __fmul_rn(lr, g.w)));
      s = m == 0 ? y
                 : make_float4(__fadd_rn(s.x, y.x), __fadd_rn(s.y, y.y), __fadd_rn(s.z, y.z), __fadd_rn(s.w, y.w));
    }
    reinterpret_cast<float4*>(out)[i] = s;
  }
  for (int64_t j = 4 * n4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
    float s = 0.f;
    for (int m = 0; m < a.m; ++m) {
      const float y = __fsub_rn(a.x[m][j], __fmul_rn(lr, a.g[m][j]));
      s = m == 0 ? y : __fadd_rn(s, y);
    }
    out[j] = s;
  }
}

// x_m = fl(s / k) for every member
__global__ void __launch_bounds__(kBThreads) scatter_mean_kernel(const float* __restrict__ s, int64_t n, float k,
                                                                 const ScatterArgs a) {
  const int64_t n4 = n / 4, stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(s) + i);
    const float4 r = make_float4(__fdiv_rn(v.x, k), __fdiv_rn(v.y, k), __fdiv_rn(v.z, k), __fdiv_rn(v.w, k));
    for (int m = 0; m < a.m; ++m) __stcs(reinterpret_cast<float4*>(a.x[m]) + i, r);
  }
  for (int64_t j = 4 * n4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
    const float r = __fdiv_rn(s[j], k);
    for (int m = 0; m < a.m; ++m) a.x[m][j] = r;
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace rp

extern "C" {

int rp_bench_presum(const float* const* x, const float* const* g, int32_t m, int64_t n, float lr, float* out,
                    void* stream) {
  if (m < 1 || m > rp::kBMax || n < 1 || !x || !g || !out || !rp::aligned16(out))
    return rp::fail(RP_EINVAL, "rp_bench_presum: 1..16 members, n >= 1, 16-byte aligned buffers");
  rp::PresumArgs a{};
  a.m = m;
  for (int i = 0; i < m; ++i) {
    if (!x[i] || !g[i] || !rp::aligned16(x[i]) || !rp::aligned16(g[i]))
      return rp::fail(RP_EINVAL, "rp_bench_presum: member buffers must be non-null and 16-byte aligned");
    a.x[i] = x[i];
    a.g[i] = g[i];
  }
  rp::presum_kernel<<<rp::grid_for(n / 4), rp::kBThreads, 0, static_cast<cudaStream_t>(stream)>>>(a, n, lr, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RP_OK : rp::fail(RP_ECUDA, std::string("rp_bench_presum: ") + cudaGetErrorString(e));
}

int rp_bench_scatter_mean(const float* s, int64_t n, float k, float* const* x, int32_t m, void* stream) {
  if (m < 1 || m > rp::kBMax || n < 1 || !s || !x || !rp::aligned16(s) || !(k > 0.f))
    return rp::fail(RP_EINVAL, "rp_bench_scatter_mean: 1..16 members, n >= 1, k > 0, 16-byte aligned buffers");
  rp::ScatterArgs a{};
  a.m = m;
  for (int i = 0; i < m; ++i) {
    if (!x[i] || !rp::aligned16(x[i])) return rp::fail(RP_EINVAL, "rp_bench_scatter_mean: misaligned member");
    a.x[i] = x[i];
  }
  rp::scatter_mean_kernel<<<rp::grid_for(n / 4), rp::kBThreads, 0, static_cast<cudaStream_t>(stream)>>>(s, n, k, a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RP_OK
                          : rp::fail(RP_ECUDA, std::string("rp_bench_scatter_mean: ") + cudaGetErrorString(e));
}

}  // extern "C"
