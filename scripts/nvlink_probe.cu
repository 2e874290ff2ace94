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
  float ms = time_kernel(0, [&] { cudaMemcpyPeerAsync(b0, 0, a1, 1, bytes); }, 10);
  printf("cudaMemcpyPeerAsync 1->0: %7.1f GB/s\n", bytes / ms / 1e6);
  ms = time_kernel(0, [&] { cudaMemcpyAsync(b0, a0, bytes, cudaMemcpyDeviceToDevice); }, 10);
  printf("local copy on GPU0: %7.1f GB/s (read+write counted once)\n", bytes / ms / 1e6);
  return 0;
}
