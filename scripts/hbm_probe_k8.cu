// HBM microbenchmark for a large group (k = 8) on one GPU: all-members-at-once loads vs a
// member-major loop (fold member by member, two streams live at a time). GB/s of 12 k N.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/hbm_probe_k8.cu -o hbm_probe_k8
#include <cuda_runtime.h>
#include <cstdio>

constexpr int K = 8;
struct Ptrs { float* x[K]; const float* g[K]; };

__device__ __forceinline__ float4 ld(const float* p) {
  float4 v;
  asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float f1(float x, float g) { return __fsub_rn(x, __fmul_rn(0.1f, g)); }
__device__ __forceinline__ float4 y4(float4 x, float4 g) { return make_float4(f1(x.x, g.x), f1(x.y, g.y), f1(x.z, g.z), f1(x.w, g.w)); }
__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w)); }
__device__ __forceinline__ float4 div4(float4 a, float k) { return make_float4(__fdiv_rn(a.x, k), __fdiv_rn(a.y, k), __fdiv_rn(a.z, k), __fdiv_rn(a.w, k)); }

template <int U>
__global__ void __launch_bounds__(256) allmem(Ptrs P, long n4) {
  for (long b = (long)blockIdx.x * 256 * U + threadIdx.x; b < n4; b += (long)gridDim.x * 256 * U) {
    float4 xv[U][K], gv[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int m = 0; m < K; ++m) { long i = b + u * 256; if (i < n4) { xv[u][m] = ld(P.x[m] + 4 * i); gv[u][m] = ld(P.g[m] + 4 * i); } }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = b + u * 256;
      if (i >= n4) continue;
      float4 s = y4(xv[u][0], gv[u][0]);
#pragma unroll
      for (int m = 1; m < K; ++m) s = add4(s, y4(xv[u][m], gv[u][m]));
      s = div4(s, (float)K);
#pragma unroll
      for (int m = 0; m < K; ++m) st(P.x[m] + 4 * i, s);
    }
  }
}

// member-major: for a tile of U float4 per thread, fold member by member (pinned order kept)
template <int U>
__global__ void __launch_bounds__(256) memmajor(Ptrs P, long n4) {
  for (long b = (long)blockIdx.x * 256 * U + threadIdx.x; b < n4; b += (long)gridDim.x * 256 * U) {
    float4 s[U];
#pragma unroll
    for (int m = 0; m < K; ++m) {
      float4 xv[U], gv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { long i = b + u * 256; if (i < n4) { xv[u] = ld(P.x[m] + 4 * i); gv[u] = ld(P.g[m] + 4 * i); } }
#pragma unroll
      for (int u = 0; u < U; ++u) s[u] = m == 0 ? y4(xv[u], gv[u]) : add4(s[u], y4(xv[u], gv[u]));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = b + u * 256;
      if (i >= n4) continue;
      const float4 r = div4(s[u], (float)K);
#pragma unroll
      for (int m = 0; m < K; ++m) st(P.x[m] + 4 * i, r);
    }
  }
}

__global__ void fill(float* p, long n, unsigned long long seed) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned long long z = seed * 0x9E3779B97F4A7C15ull + i;
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = (float)(z >> 40) * 0x1p-23f - 1.0f;
  }
}

template <typename L>
float timeit(L f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize(); cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) f();
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms / 20;
}

int main() {
  const long n = 25557032L, n4 = n / 4;
  Ptrs P;
  for (int m = 0; m < K; ++m) {
    cudaMalloc(&P.x[m], n * 4); cudaMalloc((void**)&P.g[m], n * 4);
    fill<<<1184, 256>>>(P.x[m], n, 2 * m + 1); fill<<<1184, 256>>>(const_cast<float*>(P.g[m]), n, 2 * m + 2);
  }
  cudaDeviceSynchronize();
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double algo = 12.0 * K * n;
  for (int bps : {1, 2, 4}) {
    printf("allmem U1 grid=%d: %.1f GB/s\n", sms * bps, algo / timeit([&] { allmem<1><<<sms * bps, 256>>>(P, n4); }) / 1e6);
    printf("memmajor U2 grid=%d: %.1f GB/s\n", sms * bps, algo / timeit([&] { memmajor<2><<<sms * bps, 256>>>(P, n4); }) / 1e6);
    printf("memmajor U4 grid=%d: %.1f GB/s\n", sms * bps, algo / timeit([&] { memmajor<4><<<sms * bps, 256>>>(P, n4); }) / 1e6);
    printf("memmajor U8 grid=%d: %.1f GB/s\n", sms * bps, algo / timeit([&] { memmajor<8><<<sms * bps, 256>>>(P, n4); }) / 1e6);
  }
  return 0;
}
