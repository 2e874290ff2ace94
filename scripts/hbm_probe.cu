// HBM microbenchmark for the intra-GPU P-Reduce (one GPU): the fused SGD + mean of a
// k-member group (k x's and k g's read, k x's written) in several load/store flavours,
// plus read-only and copy references. Prints GB/s of algorithmic bytes (12 k N).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/hbm_probe.cu -o hbm_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

constexpr int K = 3;
struct Ptrs {
  float* x[K];
  const float* g[K];
};

template <int MODE>
__device__ __forceinline__ float4 ldx(const float* p) {
  float4 v;
  if (MODE == 0 || MODE == 4)
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else if (MODE == 1 || MODE == 3)
    asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
template <int MODE>
__device__ __forceinline__ float4 ldg(const float* p) {
  float4 v;
  if (MODE == 0 || MODE == 4)
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else if (MODE == 1 || MODE == 3)
    asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
template <int MODE>
__device__ __forceinline__ void stx(float* p, float4 v) {
  if (MODE == 1 || MODE == 4)
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  else
    asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__device__ __forceinline__ float f1(float x, float g) { return __fsub_rn(x, __fmul_rn(0.1f, g)); }

template <int U, int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) fused(Ptrs P, long n4) {
  const long stride = (long)gridDim.x * 256 * U;
  for (long base = (long)blockIdx.x * 256 * U + threadIdx.x; base < n4; base += stride) {
    float4 xv[U][K], gv[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + u * 256;
      if (i < n4)
#pragma unroll
        for (int m = 0; m < K; ++m) {
          xv[u][m] = ldx<MODE>(P.x[m] + 4 * i);
          gv[u][m] = ldg<MODE>(P.g[m] + 4 * i);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + u * 256;
      if (i < n4) {
        float4 r;
        float s;
        s = f1(xv[u][0].x, gv[u][0].x);
        for (int m = 1; m < K; ++m) s = __fadd_rn(s, f1(xv[u][m].x, gv[u][m].x));
        r.x = __fdiv_rn(s, (float)K);
        s = f1(xv[u][0].y, gv[u][0].y);
        for (int m = 1; m < K; ++m) s = __fadd_rn(s, f1(xv[u][m].y, gv[u][m].y));
        r.y = __fdiv_rn(s, (float)K);
        s = f1(xv[u][0].z, gv[u][0].z);
        for (int m = 1; m < K; ++m) s = __fadd_rn(s, f1(xv[u][m].z, gv[u][m].z));
        r.z = __fdiv_rn(s, (float)K);
        s = f1(xv[u][0].w, gv[u][0].w);
        for (int m = 1; m < K; ++m) s = __fadd_rn(s, f1(xv[u][m].w, gv[u][m].w));
        r.w = __fdiv_rn(s, (float)K);
#pragma unroll
        for (int m = 0; m < K; ++m) stx<MODE>(P.x[m] + 4 * i, r);
      }
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

// read-only reference: sum of 2K streams
template <int U>
__global__ void __launch_bounds__(256) readonly(Ptrs P, long n4, float* out) {
  const long stride = (long)gridDim.x * 256 * U;
  float acc = 0;
  for (long base = (long)blockIdx.x * 256 * U + threadIdx.x; base < n4; base += stride) {
    float4 v[U][2 * K];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + u * 256;
      if (i < n4)
#pragma unroll
        for (int m = 0; m < K; ++m) {
          v[u][2 * m] = ldx<0>(P.x[m] + 4 * i);
          v[u][2 * m + 1] = ldg<0>(P.g[m] + 4 * i);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * 256 < n4)
#pragma unroll
        for (int m = 0; m < 2 * K; ++m) acc += v[u][m].x + v[u][m].y + v[u][m].z + v[u][m].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

template <typename L>
float timeit(L launch, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const long n = 25557032L * 8 / 3 / 4 * 4;  // ~ the bytes of one cfg2 step in one K=3 group
  const long n4 = n / 4;
  Ptrs P;
  for (int m = 0; m < K; ++m) {
    CK(cudaMalloc(&P.x[m], n * 4));
    CK(cudaMalloc((void**)&P.g[m], n * 4));
    CK(cudaMemset(P.x[m], 0, n * 4));
    CK(cudaMemset((void*)P.g[m], 0, n * 4));
  }
  float* out;
  CK(cudaMalloc(&out, 4));
  for (int m = 0; m < K; ++m) {  // non-zero, incompressible data
    fill<<<1184, 256>>>(P.x[m], n, 2 * m + 1);
    fill<<<1184, 256>>>(const_cast<float*>(P.g[m]), n, 2 * m + 2);
  }
  CK(cudaDeviceSynchronize());
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double algo = 12.0 * K * n;
  printf("n=%ld per member, algorithmic bytes per launch %.2f GB\n", n, algo / 1e9);
#define RUN(NAME, U, MODE, MINB, BPS)                                                              \
  {                                                                                                \
    int grid = sms * BPS;                                                                          \
    float ms = timeit([&] { fused<U, MODE, MINB><<<grid, 256>>>(P, n4); });                        \
    printf("%-40s grid=%5d: %8.1f GB/s  (%.3f ms)\n", NAME, grid, algo / ms / 1e6, ms);          \
  }
  RUN("U2 mode0 (current)", 2, 0, 1, 2);
  RUN("U2 mode0 4 CTAs/SM bound", 2, 0, 3, 3);
  RUN("U1 mode0", 1, 0, 1, 4);
  RUN("U1 mode0 minB4", 1, 0, 4, 4);
  RUN("U4 mode0", 4, 0, 1, 1);
  RUN("U2 mode1 (.cs loads+stores)", 2, 1, 1, 2);
  RUN("U2 mode2 (L2::256B prefetch)", 2, 2, 1, 2);
  RUN("U2 mode3 (.cs loads only)", 2, 3, 1, 2);
  RUN("U2 mode4 (.cs stores only)", 2, 4, 1, 2);
  RUN("U1 mode1 (.cs) grid x4", 1, 1, 1, 4);
  RUN("U1 mode2 minB4", 1, 2, 4, 4);
  RUN("U2 mode0 grid x8", 2, 0, 1, 8);
  {
    int grid = sms * 4;
    float ms = timeit([&] { readonly<2><<<grid, 256>>>(P, n4, out); });
    printf("%-40s grid=%5d: %8.1f GB/s read\n", "read-only 2K streams", grid, 8.0 * K * n / ms / 1e6);
  }
  {
    float ms = timeit([&] { cudaMemcpyAsync(P.x[0], P.g[0], n * 4, cudaMemcpyDeviceToDevice); });
    printf("%-40s: %8.1f GB/s (read + write)\n", "cudaMemcpy D2D", 8.0 * n / ms / 1e6);
  }
  return 0;
}
