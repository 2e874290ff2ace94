// alg1 step 2 inside the fused kernels, pinned fp32 (reading R1):
// every operation is one IEEE round-to-nearest (__fmul_rn / __fadd_rn / __fsub_rn), no FMA.
//   plain SGD:                  y = fl(x - fl(lr g))
//   momentum + weight decay     g' = fl(g + fl(wd x)); v <- fl(fl(mu v) + g'); y = fl(x - fl(lr v))
//   ("Momentum optimizer ... momentum=0.9 and weight_decay=1e-4", reading R24)
//   no staged step:             y = x
#pragma once

#include <cuda_runtime.h>

#include "rp_internal.h"

namespace rp {

__device__ __forceinline__ float step_sgd(float x, float g, float lr) { return __fsub_rn(x, __fmul_rn(lr, g)); }

__device__ __forceinline__ float step_mom(float x, float g, float& v, float lr, float mu, float wd) {
  const float gp = __fadd_rn(g, __fmul_rn(wd, x));
  v = __fadd_rn(__fmul_rn(mu, v), gp);
  return __fsub_rn(x, __fmul_rn(lr, v));
}

// One member's update of a float4: reads g (and v) that the caller loaded, returns y and,
// for momentum, the new v in `v`.
template <bool MOM>
__device__ __forceinline__ float4 step4(float4 x, float4 g, float4& v, const MemberUpdate& u) {
  if (u.g == nullptr) return x;
  if (MOM && u.v != nullptr)
    return make_float4(step_mom(x.x, g.x, v.x, u.lr, u.mu, u.wd), step_mom(x.y, g.y, v.y, u.lr, u.mu, u.wd),
                       step_mom(x.z, g.z, v.z, u.lr, u.mu, u.wd), step_mom(x.w, g.w, v.w, u.lr, u.mu, u.wd));
  return make_float4(step_sgd(x.x, g.x, u.lr), step_sgd(x.y, g.y, u.lr), step_sgd(x.z, g.z, u.lr),
                     step_sgd(x.w, g.w, u.lr));
}

// Scalar element j of one member (ragged tails): loads g / v, stores the new v.
template <bool MOM>
__device__ __forceinline__ float step1(float x, const MemberUpdate& u, int64_t j) {
  if (u.g == nullptr) return x;
  if (MOM && u.v != nullptr) {
    float v = u.v[j];
    const float y = step_mom(x, u.g[j], v, u.lr, u.mu, u.wd);
    u.v[j] = v;
    return y;
  }
  return step_sgd(x, u.g[j], u.lr);
}

}  // namespace rp
