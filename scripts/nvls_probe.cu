// NVLS (NVLink SHARP) probe, single process driving kp GPUs: is multicast supported on this
// box, and how fast is an in-switch P-Reduce (multimem.ld_reduce of a slice + multimem.st of
// the mean) of a ResNet-50-sized fp32 vector compared with the push kernel's ~500 GB/s?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvls_probe nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    CUresult r_ = (x);                                                                \
    if (r_ != CUDA_SUCCESS) {                                                         \
      const char* s_ = nullptr;                                                       \
      cuGetErrorString(r_, &s_);                                                      \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_ ? s_ : "?");    \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)
#define CR(x)                                                                         \
  do {                                                                                \
    cudaError_t r_ = (x);                                                             \
    if (r_ != cudaSuccess) {                                                          \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(r_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

template <int U>
__global__ void nvls_mean(float* mc, int64_t lo4, int64_t hi4, float kf, int divide) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = lo4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < hi4; i0 += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < hi4)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                     : "l"(mc + 4 * i)
                     : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < hi4) {
        if (divide) {
          v[u].x = __fdiv_rn(v[u].x, kf);
          v[u].y = __fdiv_rn(v[u].y, kf);
          v[u].z = __fdiv_rn(v[u].z, kf);
          v[u].w = __fdiv_rn(v[u].w, kf);
        }
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + 4 * i), "f"(v[u].x),
                     "f"(v[u].y), "f"(v[u].z), "f"(v[u].w)
                     : "memory");
      }
    }
  }
}

__global__ void fill(float* p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v + (float)(i % 7);
}

int main(int argc, char** argv) {
  const int kp = argc > 1 ? std::atoi(argv[1]) : 2;
  const int64_t n = argc > 2 ? std::atoll(argv[2]) : 25557032;
  const int ctas_per_sm = argc > 3 ? std::atoi(argv[3]) : 2;
  const int threads = argc > 4 ? std::atoi(argv[4]) : 512;
  const int unroll = argc > 5 ? std::atoi(argv[5]) : 1;
  const int gmode = argc > 6 ? std::atoi(argv[6]) : 0;  // 0 minimum, 1 recommended granularity
  CK(cuInit(0));
  int ndev = 0;
  CR(cudaGetDeviceCount(&ndev));
  if (ndev < kp) {
    std::printf("need %d GPUs, have %d\n", kp, ndev);
    return 0;
  }
  for (int d = 0; d < kp; ++d) {
    int mcs = 0;
    CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
    std::printf("dev %d multicast_supported=%d\n", d, mcs);
    if (!mcs) return 0;
  }
  CUmulticastObjectProp prop = {};
  prop.numDevices = kp;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  prop.size = n * 4;
  CK(cuMulticastGetGranularity(&gran, &prop, gmode ? CU_MULTICAST_GRANULARITY_RECOMMENDED
                                                   : CU_MULTICAST_GRANULARITY_MINIMUM));
  const size_t size = ((n * 4 + gran - 1) / gran) * gran;
  prop.size = size;
  std::printf("granularity %zu size %zu\n", gran, size);
  CUmemGenericAllocationHandle mc;
  CK(cuMulticastCreate(&mc, &prop));
  for (int d = 0; d < kp; ++d) CK(cuMulticastAddDevice(mc, d));
  std::vector<float*> uc(kp), mcp(kp);
  std::vector<cudaStream_t> st(kp);
  std::vector<cudaEvent_t> e0(kp), e1(kp);
  for (int d = 0; d < kp; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaFree(nullptr));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g2 = 0;
    CK(cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle mh;
    CK(cuMemCreate(&mh, size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mh, 0, size, 0));
    CUdeviceptr u = 0, m = 0;
    CK(cuMemAddressReserve(&u, size, gran, 0, 0));
    CK(cuMemMap(u, size, 0, mh, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(u, size, &ad, 1));
    CK(cuMemAddressReserve(&m, size, gran, 0, 0));
    CK(cuMemMap(m, size, 0, mc, 0));
    CK(cuMemSetAccess(m, size, &ad, 1));
    uc[d] = reinterpret_cast<float*>(u);
    mcp[d] = reinterpret_cast<float*>(m);
    CR(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CR(cudaEventCreate(&e0[d]));
    CR(cudaEventCreate(&e1[d]));
    fill<<<1184, 256, 0, st[d]>>>(uc[d], n, (float)(d + 1));
  }
  for (int d = 0; d < kp; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaStreamSynchronize(st[d]));
  }
  int sms = 148;
  const int64_t n4 = n / 4;
  auto run_all = [&](int divide) {
    for (int d = 0; d < kp; ++d) {
      CR(cudaSetDevice(d));
      const int64_t lo = n4 * d / kp, hi = n4 * (d + 1) / kp;
      const dim3 g(sms * ctas_per_sm);
      switch (unroll) {
        case 2: nvls_mean<2><<<g, threads, 0, st[d]>>>(mcp[d], lo, hi, (float)kp, divide); break;
        case 4: nvls_mean<4><<<g, threads, 0, st[d]>>>(mcp[d], lo, hi, (float)kp, divide); break;
        case 8: nvls_mean<8><<<g, threads, 0, st[d]>>>(mcp[d], lo, hi, (float)kp, divide); break;
        default: nvls_mean<1><<<g, threads, 0, st[d]>>>(mcp[d], lo, hi, (float)kp, divide); break;
      }
    }
  };
  run_all(1);
  for (int d = 0; d < kp; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaStreamSynchronize(st[d]));
    CR(cudaGetLastError());
  }
  // check: every GPU holds mean_d (d+1) + i%7 = (kp+1)/2 + i%7
  int bad = 0;
  for (int d = 0; d < kp; ++d) {
    std::vector<float> h(4096);
    CR(cudaSetDevice(d));
    CR(cudaMemcpy(h.data(), uc[d] + (n4 * 4 / 2), 4096 * 4, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 4096; ++i) {
      const float want = (float)(kp + 1) / 2.f + (float)((n4 * 4 / 2 + i) % 7);
      if (h[i] != want) {
        if (bad < 5) std::printf("dev %d i %d got %f want %f\n", d, i, h[i], want);
        ++bad;
      }
    }
  }
  std::printf("check: %s\n", bad ? "MISMATCH" : "ok");
  const int iters = 20;
  for (int w = 0; w < 3; ++w) run_all(0);
  for (int d = 0; d < kp; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaStreamSynchronize(st[d]));
  }
  for (int d = 0; d < kp; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaEventRecord(e0[d], st[d]));
  }
  for (int it = 0; it < iters; ++it) run_all(0);
  for (int d = 0; d < kp; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaEventRecord(e1[d], st[d]));
  }
  float worst = 0;
  for (int d = 0; d < kp; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaEventSynchronize(e1[d]));
    float ms = 0;
    CR(cudaEventElapsedTime(&ms, e0[d], e1[d]));
    if (ms > worst) worst = ms;
  }
  const double t = worst / iters / 1e3;
  const double bytes = 4.0 * n;
  std::printf("U=%d gran=%zu ", unroll, gran);
  std::printf("kp=%d n=%lld ctas/sm=%d threads=%d: %.4f ms per P-Reduce, algbw %.1f GB/s (4N/t), "
              "ring-equivalent busbw %.1f GB/s (2(kp-1)/kp*4N/t)\n",
              kp, (long long)n, ctas_per_sm, threads, t * 1e3, bytes / t / 1e9,
              2.0 * (kp - 1) / kp * bytes / t / 1e9);
  return 0;
}
