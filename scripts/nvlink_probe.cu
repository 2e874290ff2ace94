// NVLink peer-access microbenchmark (single process, GPUs 0 and 1): kernel LDG.128
// reads from the peer, kernel STG.128 writes to the peer, both directions at once,
// and cudaMemcpyPeerAsync, at several bytes-in-flight settings. Prints GB/s.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/nvlink_probe.cu -o nvlink_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e = (x);                                                                  \
    if (e != cudaSuccess) {                                                               \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

template <int U>
__global__ void peer_read(const float4* __restrict__ src, float4* __restrict__ dst, long n4) {
  long stride = (long)gridDim.x * blockDim.x * U;
  for (long base = (long)blockIdx.x * blockDim.x * U + threadIdx.x; base < n4; base += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + (long)u * blockDim.x;
      if (i < n4) v[u] = src[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + (long)u * blockDim.x;
      if (i < n4) dst[i] = v[u];
    }
  }
}

template <int U>
__global__ void peer_write(const float4* __restrict__ src, float4* __restrict__ dst, long n4) {
  long stride = (long)gridDim.x * blockDim.x * U;
  for (long base = (long)blockIdx.x * blockDim.x * U + threadIdx.x; base < n4; base += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + (long)u * blockDim.x;
      if (i < n4) v[u] = src[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long i = base + (long)u * blockDim.x;
      if (i < n4) dst[i] = v[u];
    }
  }
}

// item_A-like: read x and g locally, y = x - 0.1 g, store y to the peer; per CH float4 chunk
// (one CTA per chunk, chunks strided over the grid) optional fence.sys + flag
template <int U, bool ASM, bool FENCE>
__global__ void push_like(const float4* __restrict__ x, const float4* __restrict__ g, float4* __restrict__ dst,
                          long n4, long ch, unsigned long long* flag) {
  const long nch = (n4 + ch - 1) / ch;
  for (long c = blockIdx.x; c < nch; c += gridDim.x) {
    const long lo = c * ch, hi = min(lo + ch, n4);
    for (long t0 = lo; t0 < hi; t0 += 256 * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long i = t0 + u * 256 + threadIdx.x;
        if (i < hi) {
          float4 a, b;
          if (ASM) {
            asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "l"(x + i));
            asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "l"(g + i));
          } else {
            a = x[i];
            b = g[i];
          }
          v[u] = make_float4(a.x - 0.1f * b.x, a.y - 0.1f * b.y, a.z - 0.1f * b.z, a.w - 0.1f * b.w);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long i = t0 + u * 256 + threadIdx.x;
        if (i < hi) {
          if (ASM)
            asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i), "f"(v[u].x), "f"(v[u].y), "f"(v[u].z), "f"(v[u].w) : "memory");
          else
            dst[i] = v[u];
        }
      }
    }
    if (FENCE) {
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag + c), "l"((unsigned long long)c + 1) : "memory");
      }
    }
  }
}

template <typename K>
float time_kernel(int dev, K launch, int reps) {
  cudaSetDevice(dev);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  const long bytes = 512L << 20;
  const long n4 = bytes / 16;
  float4 *a0, *b0, *a1, *b1;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 1, bytes));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMemset(a1, 1, bytes));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("bytes per transfer %ld MiB, SMs %d\n", bytes >> 20, sms);
  for (int bpsm : {1, 2, 4, 8}) {
    const int grid = sms * bpsm;
    float ms;
    ms = time_kernel(0, [&] { peer_read<4><<<grid, 256>>>(a1, b0, n4); }, 10);
    printf("read  peer->local  grid=%4d U=4 : %7.1f GB/s\n", grid, bytes / ms / 1e6);
    ms = time_kernel(0, [&] { peer_read<8><<<grid, 256>>>(a1, b0, n4); }, 10);
    printf("read  peer->local  grid=%4d U=8 : %7.1f GB/s\n", grid, bytes / ms / 1e6);
    ms = time_kernel(0, [&] { peer_write<4><<<grid, 256>>>(a0, b1, n4); }, 10);
    printf("write local->peer  grid=%4d U=4 : %7.1f GB/s\n", grid, bytes / ms / 1e6);
  }
  // both GPUs read from each other at once (bidirectional)
  for (int bpsm : {2, 4}) {
    const int grid = sms * bpsm;
    cudaSetDevice(0);
    cudaDeviceSynchronize();
    cudaSetDevice(1);
    cudaDeviceSynchronize();
    cudaEvent_t s0, e0;
    cudaSetDevice(0);
    cudaEventCreate(&s0);
    cudaEventCreate(&e0);
    cudaEventRecord(s0);
    for (int r = 0; r < 10; ++r) {
      cudaSetDevice(0);
      peer_read<8><<<grid, 256>>>(a1, b0, n4);
      cudaSetDevice(1);
      peer_read<8><<<grid, 256>>>(a0, b1, n4);
    }
    cudaSetDevice(1);
    cudaDeviceSynchronize();
    cudaSetDevice(0);
    cudaEventRecord(e0);
    cudaEventSynchronize(e0);
    float ms;
    cudaEventElapsedTime(&ms, s0, e0);
    printf("bidir read (each GPU reads the other) grid=%d: %7.1f GB/s per direction\n", grid,
           bytes * 10 / ms / 1e6);
    cudaEventRecord(s0);
    for (int r = 0; r < 10; ++r) {
      cudaSetDevice(0);
      peer_write<4><<<grid, 256>>>(a0, b1, n4);
      cudaSetDevice(1);
      peer_write<4><<<grid, 256>>>(a1, b0, n4);
    }
    cudaSetDevice(1);
    cudaDeviceSynchronize();
    cudaSetDevice(0);
    cudaEventRecord(e0);
    cudaEventSynchronize(e0);
    cudaEventElapsedTime(&ms, s0, e0);
    printf("bidir write (each GPU writes the other) grid=%d: %7.1f GB/s per direction\n", grid,
           bytes * 10 / ms / 1e6);
  }
  {
    // item_A-like pushes, both GPUs at once (GPU0 -> GPU1 and GPU1 -> GPU0), 256 MiB each
    unsigned long long *f0, *f1;
    cudaSetDevice(0);
    cudaMalloc(&f0, 1 << 20);
    cudaSetDevice(1);
    cudaMalloc(&f1, 1 << 20);
    const long m4 = n4 / 2;
    auto both = [&](auto k0, auto k1, const char* name) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaSetDevice(0);
        cudaDeviceSynchronize();
        cudaSetDevice(1);
        cudaDeviceSynchronize();
        cudaSetDevice(0);
        cudaEvent_t s0, e0;
        cudaEventCreate(&s0);
        cudaEventCreate(&e0);
        cudaEventRecord(s0);
        for (int r = 0; r < 5; ++r) {
          cudaSetDevice(0);
          k0();
          cudaSetDevice(1);
          k1();
        }
        cudaSetDevice(1);
        cudaDeviceSynchronize();
        cudaSetDevice(0);
        cudaEventRecord(e0);
        cudaEventSynchronize(e0);
        float ms;
        cudaEventElapsedTime(&ms, s0, e0);
        if (rep == 1) printf("%-52s: %7.1f GB/s per direction\n", name, m4 * 16.0 * 5 / ms / 1e6);
      }
    };
    const int grid = sms * 2;
    for (long ch : {2048L, 8192L, 65536L}) {
      char nm[128];
      snprintf(nm, sizeof nm, "push-like C++ U4 ch=%ld nofence", ch);
      both([&] { push_like<4, false, false><<<grid, 256>>>(a0, b0, b1, m4, ch, f0); },
           [&] { push_like<4, false, false><<<grid, 256>>>(a1, b1, b0, m4, ch, f1); }, nm);
      snprintf(nm, sizeof nm, "push-like asm U4 ch=%ld nofence", ch);
      both([&] { push_like<4, true, false><<<grid, 256>>>(a0, b0, b1, m4, ch, f0); },
           [&] { push_like<4, true, false><<<grid, 256>>>(a1, b1, b0, m4, ch, f1); }, nm);
      snprintf(nm, sizeof nm, "push-like asm U4 ch=%ld fence+flag", ch);
      both([&] { push_like<4, true, true><<<grid, 256>>>(a0, b0, b1, m4, ch, f0); },
           [&] { push_like<4, true, true><<<grid, 256>>>(a1, b1, b0, m4, ch, f1); }, nm);
      snprintf(nm, sizeof nm, "push-like C++ U4 ch=%ld fence+flag", ch);
      both([&] { push_like<4, false, true><<<grid, 256>>>(a0, b0, b1, m4, ch, f0); },
           [&] { push_like<4, false, true><<<grid, 256>>>(a1, b1, b0, m4, ch, f1); }, nm);
    }
  }
  float ms = time_kernel(0, [&] { cudaMemcpyPeerAsync(b0, 0, a1, 1, bytes); }, 10);
  printf("cudaMemcpyPeerAsync 1->0: %7.1f GB/s\n", bytes / ms / 1e6);
  ms = time_kernel(0, [&] { cudaMemcpyAsync(b0, a0, bytes, cudaMemcpyDeviceToDevice); }, 10);
  printf("local copy on GPU0: %7.1f GB/s (read+write counted once)\n", bytes / ms / 1e6);
  return 0;
}
