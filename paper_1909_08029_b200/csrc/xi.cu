// Synthetic input generator and compute delay (harness kernels; not part of the method).
//
// xi(s, w, t, j) = float32(MIX(KEY) >> 40) * 2^-23 - 1, with
// KEY = s*0x9E3779B97F4A7C15 + w*0xD1B54A32D192ED03 + t*0x8CB92BA72F3D8DD7 + j (mod 2^64)
// and MIX the splitmix64 finalizer. Independent
// implementation of rp_inputs/gen.py; every step is exact in fp32, so the two
// agree bit for bit (tests/test_gpu_xi.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "rp_internal.h"

namespace rp {

__device__ __forceinline__ uint64_t xi_mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__device__ __forceinline__ float xi_value(uint64_t base, uint64_t j) {
  const uint32_t m = static_cast<uint32_t>(xi_mix(base + j) >> 40);  // 24 bits
  return __fsub_rn(__fmul_rn(__uint2float_rn(m), 0x1p-23f), 1.0f);    // exact
}

__global__ void __launch_bounds__(256) fill_xi_kernel(float* __restrict__ dst, int64_t n,
                                                      uint64_t base, uint64_t j0) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  if (aligned) {
    const int64_t n4 = n >> 2;
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const uint64_t j = j0 + 4 * static_cast<uint64_t>(i);
      float4 v;
      v.x = xi_value(base, j);
      v.y = xi_value(base, j + 1);
      v.z = xi_value(base, j + 2);
      v.w = xi_value(base, j + 3);
      d4[i] = v;
    }
    for (int64_t i = (n4 << 2) + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
      dst[i] = xi_value(base, j0 + static_cast<uint64_t>(i));
  } else {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
      dst[i] = xi_value(base, j0 + static_cast<uint64_t>(i));
  }
}

int launch_fill_xi(float* dst, int64_t n, uint64_t seed, uint64_t w, uint64_t t, uint64_t j0,
                   void* stream, std::string* err) {
  if (n < 0 || (n > 0 && !dst)) {
    *err = "rp_fill_xi: bad destination";
    return RP_EINVAL;
  }
  if (n == 0) return RP_OK;
  const uint64_t base = seed * 0x9E3779B97F4A7C15ull + w * 0xD1B54A32D192ED03ull + t * 0x8CB92BA72F3D8DD7ull;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n / 4 + 255) / 256;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 8LL * sms)));
  fill_xi_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, n, base, j0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("rp_fill_xi: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

__global__ void delay_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

int launch_delay(void* stream, int64_t ns, std::string* err) {
  if (ns < 0) {
    *err = "rp_compute_delay: negative duration";
    return RP_EINVAL;
  }
  if (ns == 0) return RP_OK;
  delay_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<unsigned long long>(ns));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("rp_compute_delay: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

}  // namespace rp
