// NVLS P-Reduce: alg1 steps 2 + 4 for groups spanning several GPUs,
// with the sum over GPUs computed INSIDE the NVSwitch.
//
// The GPUs of a group share a slot of a multicast object (nvls_setup.cpp): every GPU has
// its own copy of the slot (unicast address `uc`), and a store or reduction through the
// multicast address `mc` reaches all copies. Per chunk c of the vector (CH float4):
//   P(c)  every GPU: y_m = step2(x_m, g_m) for its local members, partial = left fold
//         (ascending worker id, reading R1) -> uc[c]; then arrive[c][me] = tag on all
//         copies (multimem.st.release).
//   R(c)  the owner (position c mod kp): wait for arrive[c][*]; sum = multimem.ld_reduce
//         .add over the kp copies (in-switch); xbar = fl(sum / |G|); multimem.st xbar to
//         every copy; its own local members' x <- xbar; done[c] = tag on all copies.
//   S(c)  every non-owner: wait for done[c]; x_m <- uc[c] for its local members.
// One launch per GPU and step holds every NVLS group of the step. By default half of the
// CTAs walk the HBM items (all P, then all S) and the other half the R items, so the
// in-switch reductions overlap the HBM passes of other chunks (RP_NVLS_HBM_PCT; 0 = one
// list P*, R*, S* for every CTA). A CTA finishes its non-blocking items before it can
// block; the grid never exceeds the resident CTA count (as in xgpu.cu).
// The in-switch summation order over the kp partials is the switch's (reading R25).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "rp_internal.h"
#include "update.cuh"

namespace rp {

namespace {

constexpr int kNThreads = 256;
constexpr int kNU = 4;  // float4 per thread in flight (P and S items)

__device__ __forceinline__ float4 ldv(const float* p) {
  float4 v;
  asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ldg_nc(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void stv(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 mm_ld_reduce4(const float* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
__device__ __forceinline__ float mm_ld_reduce1(const float* mc) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st4(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st1(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}
__device__ __forceinline__ void mm_st_release_u64(unsigned long long* mc, unsigned long long v) {
  asm volatile("multimem.st.release.sys.global.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Watchdog: a peer that never posts its flag (a crashed rank, a broken collective contract) ends
// the wait after p.watchdog_ns (rp_config.watchdog_s / RP_WATCHDOG_S; 0 = wait forever): the flag
// is recorded in host-mapped memory (the host reports RP_ETIMEOUT) and every later wait of the
// job returns at once, so the kernel finishes (with garbage) instead of hanging the GPU.
__device__ __noinline__ void wait_flag(const NPart& p, const unsigned long long* f, unsigned long long tag, int kind,
                                       int64_t c) {
  if (ld_acquire_sys(f) == tag) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (unsigned n = 1; ld_acquire_sys(f) != tag; ++n) {
    __nanosleep(32);
    if (p.watchdog_ns && (n & 1023u) == 0) {
      if (p.err && *reinterpret_cast<volatile unsigned long long*>(&p.err->code)) return;  // job already failed
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > p.watchdog_ns) {
        if (p.err && atomicCAS(&p.err->code, 0ull, 1ull) == 0ull) {
          p.err->gpu = p.gpu;
          p.err->src = -1;
          p.err->kind = 16 + kind;  // NVLS flag kinds
          p.err->slot = -1;
          p.err->chunk = c;
          p.err->tag = tag;
          p.err->seen = ld_acquire_sys(f);
          __threadfence_system();
        }
        return;
      }
    }
  }
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 div4(float4 a, float k) {
  return make_float4(__fdiv_rn(a.x, k), __fdiv_rn(a.y, k), __fdiv_rn(a.z, k), __fdiv_rn(a.w, k));
}

// Local partial at float4 index i: step 2 of every local member, left fold (reading R1).
template <int M, bool MOM>
__device__ __forceinline__ float4 partial4(const NPart& p, int64_t i) {
  float4 xv[M], gv[M], vv[MOM ? M : 1];
#pragma unroll
  for (int m = 0; m < M; ++m)
    if (m < p.m) {
      xv[m] = ldv(p.x[m] + 4 * i);
      if (p.u[m].g) gv[m] = ldg_nc(p.u[m].g + 4 * i);
      if constexpr (MOM)
        if (p.u[m].v) vv[m] = ldv(p.u[m].v + 4 * i);
    }
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int m = 0; m < M; ++m)
    if (m < p.m) {
      float4 vm = vv[MOM ? m : 0];
      const float4 y = step4<MOM>(xv[m], gv[m], vm, p.u[m]);
      if constexpr (MOM)
        if (p.u[m].v && p.u[m].g) stv(p.u[m].v + 4 * i, vm);
      s = m == 0 ? y : add4(s, y);
    }
  return s;
}
template <int M, bool MOM>
__device__ __forceinline__ float partial1(const NPart& p, int64_t j) {
  float s = step1<MOM>(p.x[0][j], p.u[0], j);
#pragma unroll
  for (int m = 1; m < M; ++m)
    if (m < p.m) s = __fadd_rn(s, step1<MOM>(p.x[m][j], p.u[m], j));
  return s;
}

// flags of chunk c: arrive[0..7], done
__device__ __forceinline__ int64_t fl_arrive(int64_t c, int pos) { return c * kNvlsFlagStride + pos; }
__device__ __forceinline__ int64_t fl_done(int64_t c) { return c * kNvlsFlagStride + 8; }

// post a flag on every copy after all of this CTA's prior stores
__device__ __forceinline__ void post(unsigned long long* mcf, int64_t idx, unsigned long long tag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    mm_st_release_u64(mcf + idx, tag);
  }
}
__device__ __forceinline__ void await(const NPart& p, const unsigned long long* ucf, int64_t idx, unsigned long long tag,
                                      int64_t c) {
  if (threadIdx.x == 0) wait_flag(p, ucf + idx, tag, 1, c);
  __syncthreads();
}

template <int M, bool MOM>
__device__ void item_P(const NPart& p, int64_t c) {
  const int64_t lo = c * p.CH, hi = min(lo + p.CH, p.n4);
  for (int64_t t0 = lo; t0 < hi; t0 += kNThreads * kNU) {
    float4 s[kNU];
#pragma unroll
    for (int u = 0; u < kNU; ++u) {
      const int64_t i = t0 + u * kNThreads + threadIdx.x;
      if (i < hi) s[u] = partial4<M, MOM>(p, i);
    }
#pragma unroll
    for (int u = 0; u < kNU; ++u) {
      const int64_t i = t0 + u * kNThreads + threadIdx.x;
      if (i < hi) stv(p.uc + 4 * i, s[u]);
    }
  }
  if (c == p.nch - 1 && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    p.uc[j] = partial1<M, MOM>(p, j);
  }
  post(p.mcf, fl_arrive(c, p.me), p.tag);
}

template <int M>
__device__ void item_R(const NPart& p, int64_t c) {
  if (threadIdx.x == 0)
    for (int d = 0; d < p.kp; ++d) wait_flag(p, p.ucf + fl_arrive(c, d), p.tag, 0, c);
  __syncthreads();
  const int64_t lo = c * p.CH, hi = min(lo + p.CH, p.n4);
  const float kf = static_cast<float>(p.k_total);
  for (int64_t i = lo + threadIdx.x; i < hi; i += kNThreads) {
    const float4 xbar = div4(mm_ld_reduce4(p.mc + 4 * i), kf);
    mm_st4(p.mc + 4 * i, xbar);
#pragma unroll
    for (int m = 0; m < M; ++m)
      if (m < p.m) stv(p.x[m] + 4 * i, xbar);
  }
  if (c == p.nch - 1 && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    const float xbar = __fdiv_rn(mm_ld_reduce1(p.mc + j), kf);
    mm_st1(p.mc + j, xbar);
    for (int m = 0; m < p.m; ++m) p.x[m][j] = xbar;
  }
  post(p.mcf, fl_done(c), p.tag);
}

template <int M>
__device__ void item_S(const NPart& p, int64_t c) {
  await(p, p.ucf, fl_done(c), p.tag, c);
  const int64_t lo = c * p.CH, hi = min(lo + p.CH, p.n4);
  for (int64_t t0 = lo; t0 < hi; t0 += kNThreads * kNU) {
    float4 v[kNU];
#pragma unroll
    for (int u = 0; u < kNU; ++u) {
      const int64_t i = t0 + u * kNThreads + threadIdx.x;
      if (i < hi) v[u] = ldv(p.uc + 4 * i);
    }
#pragma unroll
    for (int u = 0; u < kNU; ++u) {
      const int64_t i = t0 + u * kNThreads + threadIdx.x;
      if (i < hi)
#pragma unroll
        for (int m = 0; m < M; ++m)
          if (m < p.m) stv(p.x[m] + 4 * i, v[u]);
    }
  }
  if (c == p.nch - 1 && threadIdx.x < p.rem) {
    const int64_t j = 4 * p.n4 + threadIdx.x;
    const float v = p.uc[j];
    for (int m = 0; m < p.m; ++m) p.x[m][j] = v;
  }
}

// Owned chunks of position me: me, me + kp, ...; the s-th non-owned chunk.
__device__ __forceinline__ int64_t owned_chunk(const NPart& p, int64_t r) { return p.me + r * p.kp; }
__device__ __forceinline__ int64_t other_chunk(const NPart& p, int64_t s) {
  const int64_t q = s / (p.kp - 1), r = s % (p.kp - 1);
  return q * p.kp + (r < p.me ? r : r + 1);
}

// Item q of the HBM list (P items of every part, then S items) or of the switch list (R items).
template <int M, bool MOM>
__device__ __forceinline__ void run_item(const NTask& T, int64_t q) {
  int pi = 0, phase = 0;
  int64_t k = 0;
  for (int a = T.nparts - 1; a >= 0; --a) {
    const NPart& p = T.part[a];
    if (q >= p.off_S && q < p.off_S + (p.nch - p.nown)) { phase = 2; pi = a; k = q - p.off_S; break; }
    if (q >= p.off_R && q < p.off_R + p.nown) { phase = 1; pi = a; k = q - p.off_R; break; }
    if (q >= p.off_P && q < p.off_P + p.nch) { phase = 0; pi = a; k = q - p.off_P; break; }
  }
  const NPart& p = T.part[pi];
  if (phase == 0) item_P<M, MOM>(p, k);
  else if (phase == 1) item_R<M>(p, owned_chunk(p, k));
  else item_S<M>(p, other_chunk(p, k));
}

// CTAs [0, T.hbm_ctas) walk the HBM list (all P items, then all S items); the others walk
// the switch list (R items), so in-switch reductions overlap the HBM work of other chunks.
// Without a split (hbm_ctas == 0) every CTA walks P*, R*, S* in one list. Either way a
// CTA's non-blocking items come before its blocking ones, and R waits only on P items,
// S only on R items.
template <int M, bool MOM>
__global__ void __launch_bounds__(kNThreads) nvls_kernel(const NTask T) {
  if (T.hbm_ctas == 0) {
    for (int64_t q = blockIdx.x; q < T.total_items; q += gridDim.x) run_item<M, MOM>(T, q);
    return;
  }
  if (static_cast<int>(blockIdx.x) < T.hbm_ctas) {
    for (int64_t j = blockIdx.x; j < T.n_hbm; j += T.hbm_ctas) {
      const int64_t q = j < T.n_p ? j : T.off_s0 + (j - T.n_p);  // P items, then S items
      run_item<M, MOM>(T, q);
    }
  } else {
    const int64_t g = gridDim.x - T.hbm_ctas;
    for (int64_t j = blockIdx.x - T.hbm_ctas; j < T.n_r; j += g) run_item<M, MOM>(T, T.n_p + j);
  }
}

int g_nsms = 0;

template <int M, bool MOM>
int launch_nm(NTask& T, cudaStream_t stream, std::string* err) {
  static int occ = 0;
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nvls_kernel<M, MOM>, kNThreads, 0) != cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  if (g_nsms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_nsms, cudaDevAttrMultiProcessorCount, dev);
    if (g_nsms <= 0) g_nsms = 148;
  }
  const int64_t cap = static_cast<int64_t>(g_nsms) * occ;  // all CTAs co-resident
  static int split = -1;  // percent of the CTAs on the HBM list; 0 = one list
  if (split < 0) {
    const char* v = std::getenv("RP_NVLS_HBM_PCT");
    split = v && *v ? std::atoi(v) : 50;
  }
  int blocks = static_cast<int>(std::max<int64_t>(1, std::min(cap, T.total_items)));
  T.hbm_ctas = 0;
  if (split > 0 && split < 100 && cap >= 2) {
    blocks = static_cast<int>(cap);
    T.hbm_ctas = std::max(1, std::min(blocks - 1, static_cast<int>(cap * split / 100)));
  }
  nvls_kernel<M, MOM><<<blocks, kNThreads, 0, stream>>>(T);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("nvls kernel launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

}  // namespace

int64_t nvls_chunk_f4() {
  static int64_t ch = 0;
  if (ch == 0) {
    const char* v = std::getenv("RP_NVLS_CHUNK_F4");
    ch = v && *v ? std::atoll(v) : 4096;  // 64 KiB chunks
    ch = std::max<int64_t>(kNThreads * kNU, ch / (kNThreads * kNU) * (kNThreads * kNU));
  }
  return ch;
}

int launch_nvls(NTask& T, void* stream, std::string* err) {
  if (T.nparts < 1 || T.nparts > kMaxNParts) {
    *err = "nvls: bad part count";
    return RP_EINVAL;
  }
  int mmax = 0;
  bool mom = false;
  int64_t off = 0;
  for (int pi = 0; pi < T.nparts; ++pi) {
    NPart& p = T.part[pi];
    if (p.m < 1 || p.m > kMaxXLocal || p.kp < 2 || p.kp > 8 || p.me < 0 || p.me >= p.kp || !p.uc || !p.mc ||
        !p.ucf || !p.mcf || p.nch < 1) {
      *err = "nvls: bad part descriptor";
      return RP_EINVAL;
    }
    mmax = std::max(mmax, p.m);
    for (int m = 0; m < p.m; ++m) mom = mom || (p.u[m].v && p.u[m].g);
    p.nown = p.nch > p.me ? (p.nch - p.me + p.kp - 1) / p.kp : 0;
    p.off_P = off;
    off += p.nch;
  }
  for (int pi = 0; pi < T.nparts; ++pi) {
    T.part[pi].off_R = off;
    off += T.part[pi].nown;
  }
  for (int pi = 0; pi < T.nparts; ++pi) {
    T.part[pi].off_S = off;
    off += T.part[pi].nch - T.part[pi].nown;
  }
  T.total_items = off;
  T.n_p = T.part[0].off_R;                    // P items: [0, n_p)
  T.n_r = T.part[0].off_S - T.n_p;            // R items: [n_p, off_s0)
  T.off_s0 = T.part[0].off_S;                 // S items: [off_s0, total)
  T.n_hbm = T.n_p + (T.total_items - T.off_s0);
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mom) {
    if (mmax <= 1) return launch_nm<1, true>(T, s, err);
    if (mmax <= 2) return launch_nm<2, true>(T, s, err);
    if (mmax <= 4) return launch_nm<4, true>(T, s, err);
    return launch_nm<8, true>(T, s, err);
  }
  if (mmax <= 1) return launch_nm<1, false>(T, s, err);
  if (mmax <= 2) return launch_nm<2, false>(T, s, err);
  if (mmax <= 4) return launch_nm<4, false>(T, s, err);
  return launch_nm<8, false>(T, s, err);
}

}  // namespace rp
