// NVLink push microbenchmark for the cross-GPU kernel's store/signal pattern (round 2).
// GPUs 0 and 1 push to each other at once (bidirectional). Each CTA owns a contiguous range,
// cut into chunks of K tiles (16 KB); per tile: y = x - 0.1 g from local HBM -> shared memory
// ring (NBUF tiles) -> TMA bulk store (cp.async.bulk global <- shared::cta) into the peer.
// Per chunk a flag is published in one of several ways:
//   mode 0  no flags (upper bound)
//   mode 1  drain: wait_group 0, fence.proxy.async, fence.sc.sys, st.release.sys flag
//   mode 2  deferred: after committing chunk c, wait until only chunk c's groups are pending
//           (wait_group K), then fence + flag for chunk c-1 (stores keep flowing meanwhile)
//   mode 3  deferred like 2, release store only (no separate fence.sc.sys)
//   mode 4  plain st.global.v4 peer stores (no smem, no TMA), drain fence + flag per chunk
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/bulk_push_probe.cu -o build/bulk_push_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

constexpr int T = 256;
constexpr int TILE = 1024;  // float4 per tile (16 KB)

__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(src));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(s), "r"(bytes) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void wait_n(int k) {
  // wait_group takes an immediate: the few values used
  switch (k) {
    case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
    case 8: asm volatile("cp.async.bulk.wait_group 8;" ::: "memory"); break;
    case 16: asm volatile("cp.async.bulk.wait_group 16;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
  }
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int NBUF>
__global__ void __launch_bounds__(T) push(const float4* __restrict__ x, const float4* __restrict__ g, float4* dst,
                                          long n4, int K, int mode, unsigned long long* flags) {
  extern __shared__ float4 sm[];
  const long per = (n4 + gridDim.x - 1) / gridDim.x;
  const long lo = blockIdx.x * per, hi = min(lo + per, n4);
  const long chunk = static_cast<long>(K) * TILE;
  int slot = 0;
  long c_idx = 0;
  for (long c0 = lo; c0 < hi; c0 += chunk, ++c_idx) {
    const long c1 = min(c0 + chunk, hi);
    for (long t0 = c0; t0 < c1; t0 += TILE) {
      if (mode == 4) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          long i = t0 + r * T + threadIdx.x;
          if (i < c1) {
            float4 a = __ldcs(x + i), b = __ldcs(g + i);
            dst[i] = make_float4(a.x - 0.1f * b.x, a.y - 0.1f * b.y, a.z - 0.1f * b.z, a.w - 0.1f * b.w);
          }
        }
        continue;
      }
      if (threadIdx.x == 0) wait_read<NBUF - 1>();
      __syncthreads();
      float4* b = sm + (slot % NBUF) * TILE;
      ++slot;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        long i = t0 + r * T + threadIdx.x;
        if (i < c1) {
          float4 a = __ldcs(x + i), gg = __ldcs(g + i);
          b[r * T + threadIdx.x] = make_float4(a.x - 0.1f * gg.x, a.y - 0.1f * gg.y, a.z - 0.1f * gg.z, a.w - 0.1f * gg.w);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        bulk_store(dst + t0, b, static_cast<unsigned>(min(static_cast<long>(TILE), c1 - t0) * 16));
        commit();
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long* f = flags + blockIdx.x * 64 + (c_idx & 63);
      if (mode == 1 || mode == 4) {
        if (mode == 1) {
          wait_all();
          asm volatile("fence.proxy.async;" ::: "memory");
        }
        __threadfence_system();
        st_release(f, c_idx + 1);
      } else if ((mode == 2 || mode == 3) && c_idx > 0) {
        const int kt = static_cast<int>((c1 - c0 + TILE - 1) / TILE);  // groups of this chunk
        wait_n(kt);
        asm volatile("fence.proxy.async;" ::: "memory");
        if (mode == 2) __threadfence_system();
        st_release(f - 1 + (c_idx & 63 ? 0 : 64), c_idx);
      }
    }
  }
  if (threadIdx.x == 0 && mode != 4) {
    wait_all();
    asm volatile("fence.proxy.async;" ::: "memory");
    __threadfence_system();
    if (mode != 0) st_release(flags + blockIdx.x * 64 + 63, ~0ull);
  }
}

// granularity: each 16 KB tile pushed as `split` bulk stores of 16/split KB (issued by thread 0)
__global__ void __launch_bounds__(T) push_split(const float4* __restrict__ x, const float4* __restrict__ g,
                                                float4* dst, long n4, int split) {
  extern __shared__ float4 sm[];
  const long per = (n4 + gridDim.x - 1) / gridDim.x;
  const long lo = blockIdx.x * per, hi = min(lo + per, n4);
  int slot = 0;
  for (long t0 = lo; t0 < hi; t0 += TILE) {
    if (threadIdx.x == 0) wait_read<2>();
    __syncthreads();
    float4* b = sm + (slot % 3) * TILE;
    ++slot;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      long i = t0 + r * T + threadIdx.x;
      if (i < hi) {
        float4 a = __ldcs(x + i), gg = __ldcs(g + i);
        b[r * T + threadIdx.x] = make_float4(a.x - 0.1f * gg.x, a.y - 0.1f * gg.y, a.z - 0.1f * gg.z, a.w - 0.1f * gg.w);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const long cnt = min(static_cast<long>(TILE), hi - t0);
      const long piece = (cnt + split - 1) / split;
      for (long q = 0; q < cnt; q += piece)
        bulk_store(dst + t0 + q, b + q, static_cast<unsigned>(min(piece, cnt - q) * 16));
      commit();
    }
  }
  if (threadIdx.x == 0) wait_all();
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("needs 2 GPUs\n");
    return 1;
  }
  const long bytes = 256L << 20, n4 = bytes / 16;
  float4 *x[2], *g[2], *d[2];
  unsigned long long* fl[2];
  cudaStream_t st[2];
  for (int i = 0; i < 2; ++i) {
    CK(cudaSetDevice(i));
    CK(cudaDeviceEnablePeerAccess(1 - i, 0));
    CK(cudaMalloc(&x[i], bytes));
    CK(cudaMalloc(&g[i], bytes));
    CK(cudaMalloc(&d[i], bytes));
    CK(cudaMalloc(&fl[i], 4096 * 64 * 8));
    CK(cudaMemset(x[i], 0, bytes));
    CK(cudaMemset(g[i], 0, bytes));
    CK(cudaStreamCreate(&st[i]));
    CK(cudaFuncSetAttribute(push<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * TILE * 16));
    CK(cudaFuncSetAttribute(push<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * TILE * 16));
  }
  CK(cudaSetDevice(0));
  CK(cudaFuncSetAttribute(push_split, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * TILE * 16));
  CK(cudaSetDevice(1));
  CK(cudaFuncSetAttribute(push_split, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * TILE * 16));
  for (int split : {1, 2, 4, 8, 16, 32}) {
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t e0[2], e1[2];
      for (int i = 0; i < 2; ++i) {
        CK(cudaSetDevice(i));
        CK(cudaEventCreate(&e0[i]));
        CK(cudaEventCreate(&e1[i]));
        CK(cudaEventRecord(e0[i], st[i]));
        push_split<<<296, T, 3 * TILE * 16, st[i]>>>(x[i], g[i], d[1 - i], n4, split);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1[i], st[i]));
      }
      float ms = 0;
      for (int i = 0; i < 2; ++i) {
        CK(cudaSetDevice(i));
        CK(cudaEventSynchronize(e1[i]));
        float m = 0;
        CK(cudaEventElapsedTime(&m, e0[i], e1[i]));
        ms = m > ms ? m : ms;
      }
      if (rep > 0 && ms < best) best = ms;
    }
    printf("granularity: 16 KB tile as %2d bulk stores of %5.2f KB  %7.1f GB/s per direction (grid 296, no flags)\n",
           split, 16.0 / split, bytes / (best * 1e-3) / 1e9);
  }
  if (getenv("PROBE_ONLY_SPLIT")) return 0;
  const char* names[] = {"no flags", "drain+fence+flag", "deferred fence+flag", "deferred release-only",
                         "plain STG drain"};
  for (int nbuf : {3, 4}) {
    for (int grid : {148, 296, 444}) {
      if (nbuf == 4 && grid == 444) continue;
      for (int K : {2, 4, 8, 16}) {
        for (int mode = 0; mode < 5; ++mode) {
          if (mode == 4 && nbuf == 4) continue;
          float best = 1e9f;
          for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0[2], e1[2];
            for (int i = 0; i < 2; ++i) {
              CK(cudaSetDevice(i));
              CK(cudaEventCreate(&e0[i]));
              CK(cudaEventCreate(&e1[i]));
            }
            for (int i = 0; i < 2; ++i) {
              CK(cudaSetDevice(i));
              CK(cudaEventRecord(e0[i], st[i]));
              if (nbuf == 3)
                push<3><<<grid, T, 3 * TILE * 16, st[i]>>>(x[i], g[i], d[1 - i], n4, K, mode, fl[1 - i]);
              else
                push<4><<<grid, T, 4 * TILE * 16, st[i]>>>(x[i], g[i], d[1 - i], n4, K, mode, fl[1 - i]);
              CK(cudaGetLastError());
              CK(cudaEventRecord(e1[i], st[i]));
            }
            float ms = 0;
            for (int i = 0; i < 2; ++i) {
              CK(cudaSetDevice(i));
              CK(cudaEventSynchronize(e1[i]));
              float m = 0;
              CK(cudaEventElapsedTime(&m, e0[i], e1[i]));
              ms = m > ms ? m : ms;
              cudaEventDestroy(e0[i]);
              cudaEventDestroy(e1[i]);
            }
            if (rep > 0 && ms < best) best = ms;
          }
          printf("nbuf=%d grid=%3d chunk=%2d tiles (%4d KB) %-24s %7.1f GB/s per direction\n", nbuf, grid, K, K * 16,
                 names[mode], bytes / (best * 1e-3) / 1e9);
        }
      }
    }
  }
  return 0;
}
