// Cross-GPU fused SGD + P-Reduce, warp-specialized (default for plain-SGD steps, fp32 and bf16).
//
// Same method, chunk geometry and flag words as xgpu.cu (read its header first): a group on GPUs
// d_0 < ... < d_{kp-1} is a reduce-scatter + all-gather fused with alg1 step 2 and the
// pre-reduction of co-resident members (reading R1). By default CTAs claim chunks dynamically and
// run the iteration structure described under "Flags" below; without a claim counter chunk c
// runs on lane c mod kXLanes in xgpu.cu's static lane pipeline.
//
// What changes is how a CTA moves the bytes. Round 2 measured the LDG/STG version per CTA
// (RP_XGPU_PROFILE breakdown, profiles/r02/): 65-96 % of a CTA's time went to loading x, g and
// the staged partials and folding them, < 2 % to waiting for its NVLink pushes -- the pushes
// were starved by the loads. Here one producer warp streams every operand tile of the lane's
// work into an S-stage shared-memory ring with TMA bulk loads (cp.async.bulk global ->
// shared, completion on the stage's `full` mbarrier), waiting for the peers' flags before a
// stage that needs their data; eight consumer warps fold each stage into an output tile and
// push it with TMA bulk stores (to the owner's staging for A, to the local members and every
// peer's first member for B, to the other local members for C), then release the stage on its
// `empty` mbarrier. Loads, arithmetic and NVLink pushes of different tiles overlap.
//
// Flags (deferred): flags are posted by SIG jobs in the stage stream. At a SIG each consumer
// warp waits until only its bulk groups committed since the previous SIG are pending (so
// everything before the previous SIG has completed), makes them visible to the generic proxy and
// arrives on a shared counter with acq_rel; the last warp releases at system scope and posts the
// flags the SIG carries. Default (dynamic chunk claiming), iteration i of a CTA: A(claim i),
// SIG_a (B flags of iteration i-1), B(claim i-1) with SIG_m after its first tile (A flags of
// claim i), C(claim i-2), fused intra-GPU tiles, SIG_b (delimiter). The static-lane fallback keeps
// xgpu.cu's lane pipeline. A wait for a peer's flag (producer warp) past the watchdog limit
// records it in host-mapped memory and ends the CTA's work (an END job lets the consumers out).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "rp_internal.h"
#include "update.cuh"

namespace rp {
namespace {

constexpr int kWarps = 8;                       // consumer warps
constexpr int kWsT = 32 * (kWarps + 1);         // + one producer warp
constexpr int kT = 512;                         // vectors per tile (8 KB per fp32 operand)
constexpr int kPW = kT / kWarps;                // vectors per consumer warp and tile
constexpr int kVPL = kPW / 32;                  // vectors per lane and tile
constexpr int kGeomTile = 1024;                 // xgpu.cu's chunk / slice alignment (vectors)
constexpr int kSigRing = 8;                     // SIG counters (> max stages)
constexpr int kJA = 0, kJB = 1, kJC = 2, kJSig = 3, kJEnd = 4, kJL = 5;

struct Job {                // one stage's work, written by the producer next to the stage
  int32_t kind, pi, o, cnt;
  int64_t base;             // first vector of the tile (absolute index in the replica)
  int64_t pA, pB;           // SIG: chunks whose flags to post
  int32_t tail;             // the chunk's n mod 4 scalar tail rides on this job
  int32_t sig;              // SIG sequence number
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_pending(int n) {
  switch (n < 63 ? n : 63) {
#define RP_W(k) \
  case k: asm volatile("cp.async.bulk.wait_group " #k ";" ::: "memory"); break;
#define RP_W8(k) RP_W(k) RP_W(k + 1) RP_W(k + 2) RP_W(k + 3) RP_W(k + 4) RP_W(k + 5) RP_W(k + 6) RP_W(k + 7)
    RP_W8(0) RP_W8(8) RP_W8(16) RP_W8(24) RP_W8(32) RP_W8(40) RP_W8(48) RP_W8(56)
#undef RP_W8
#undef RP_W
  }
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int atom_add_acq_rel_cta(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.s32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 div4(float4 a, float k) {
  return make_float4(__fdiv_rn(a.x, k), __fdiv_rn(a.y, k), __fdiv_rn(a.z, k), __fdiv_rn(a.w, k));
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t bf_rn(float v) {  // IEEE round-to-nearest-even; NaN stays NaN
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v)));
}
__device__ __forceinline__ uint2 pack_bf4(float4 v) {
  return make_uint2(bf_rn(v.x) | (bf_rn(v.y) << 16), bf_rn(v.z) | (bf_rn(v.w) << 16));
}
__device__ __forceinline__ float4 unpack_bf4(uint2 w) { return make_float4(bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y)); }

// flag word of (slot, src GPU, kind, chunk) in a GPU's flag array (layout of xgpu.cu)
__device__ __forceinline__ unsigned long long* flag_at(unsigned long long* base, int slot, int src, int kind,
                                                       int64_t c) {
  return base + (static_cast<int64_t>(slot) * kFlagSrc + src) * kFlagStride +
         (kind == kFlagA ? c : (kind == kFlagB ? kMaxChunks + c : 2 * kMaxChunks));
}

__device__ __noinline__ bool wait_flag_slow(const XTask& T, const unsigned long long* f, unsigned long long tag,
                                            int slot, int src, int kind, int64_t c) {
  const unsigned long long t0 = gtimer();
  for (unsigned n = 1;; ++n) {
    __nanosleep(32);
    if (ld_acquire_sys(f) == tag) return true;
    if (T.watchdog_ns && (n & 1023u) == 0) {
      if (T.err && *reinterpret_cast<volatile unsigned long long*>(&T.err->code)) return false;  // job failed
      if (gtimer() - t0 <= T.watchdog_ns) continue;
      if (T.err && atomicCAS(&T.err->code, 0ull, 1ull) == 0ull) {
        T.err->gpu = T.my_gpu;
        T.err->src = src;
        T.err->kind = kind;
        T.err->slot = slot;
        T.err->chunk = c;
        T.err->tag = tag;
        T.err->seen = ld_acquire_sys(f);
        __threadfence_system();
      }
      return false;
    }
  }
}
__device__ __forceinline__ bool wait_flag(const XTask& T, const unsigned long long* f, unsigned long long tag,
                                          int slot, int src, int kind, int64_t c) {
  if (ld_acquire_sys(f) == tag) return true;
  const unsigned long long t0 = T.cta_stat ? gtimer() : 0;
  const bool ok = wait_flag_slow(T, f, tag, slot, src, kind, c);
  if (T.cta_stat) {
    const unsigned long long t1 = gtimer();
    atomicAdd(T.cta_stat + 4 * blockIdx.x + 2, t1 - t0);
    const unsigned long long q = T.cta_stat[kCtaCntBase + 2 * blockIdx.x + 1]++;  // producer lane only
    if (q < kCtaWait) {
      unsigned long long* r = T.cta_stat + kCtaWaitBase + (2 * kCtaWait) * blockIdx.x + 2 * q;
      r[0] = (t0 & ~3ull) | static_cast<unsigned>(kind & 3);
      r[1] = t1;
    }
  }
  return ok;
}

struct Range {
  int64_t lo, hi;
  bool tail;
};
__device__ __forceinline__ int64_t slice_lo(const XPart& p, int o) { return min(static_cast<int64_t>(o) * p.S4, p.n4); }
__device__ __forceinline__ Range chunk_range(const XPart& p, int o, int64_t c) {
  const int64_t slo = slice_lo(p, o), shi = min(static_cast<int64_t>(o + 1) * p.S4, p.n4);
  Range r;
  // balanced big chunks: tiles [c CH / nbig, (c+1) CH / nbig); then nsmall chunks of tail_w tiles
  const int64_t nbig = p.nch - p.nsmall;
  const int64_t t_lo = c < nbig ? (c * p.CH) / nbig : p.CH + (c - nbig) * p.tail_w;
  const int64_t t_hi = c < nbig ? ((c + 1) * p.CH) / nbig : t_lo + p.tail_w;
  r.lo = min(slo + t_lo * 1024, shi);
  r.hi = min(slo + t_hi * 1024, shi);
  r.tail = (o == p.kp - 1) && (c == p.nch - 1) && p.rem > 0;
  return r;
}
__device__ __forceinline__ int64_t stage_off(const XPart& p, int d, int64_t i_rel) {
  return (static_cast<int64_t>(d) * (p.S4 + 1) + i_rel) * 4;
}

// ---- scalar tails (n mod 4 elements; plain global loads / stores, warp 0 of the consumers) ----
template <bool BF>
__device__ __forceinline__ float ldx1(const float* base, int64_t j) {
  if constexpr (BF) return __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(base)[j]) << 16);
  else return base[j];
}
template <bool BF>
__device__ __forceinline__ void stx1(float* base, int64_t j, float v) {
  if constexpr (BF) reinterpret_cast<uint16_t*>(base)[j] = static_cast<uint16_t>(bf_rn(v));
  else base[j] = v;
}
template <int M, bool BF>
__device__ __forceinline__ float partial1(const XPart& p, int64_t j) {
  float s = 0.f;
#pragma unroll
  for (int m = 0; m < M; ++m)
    if (m < p.m) {
      float y = ldx1<BF>(p.x[m], j);
      if (p.u[m].g) y = step_sgd(y, ldx1<BF>(p.u[m].g, j), p.u[m].lr);
      s = m == 0 ? y : __fadd_rn(s, y);
    }
  return s;
}

// Shared-memory layout: S stages of NOP operand slots of kT vectors (16 bytes per vector per slot,
// bf16 operands use the first half), the output tiles [2][kT], S full + S empty mbarriers,
// S job descriptors, the SIG counters and the abort word.
template <int NOP, int S>
constexpr size_t ws_smem() {
  return static_cast<size_t>(S) * NOP * kT * 16 + 2 * kT * 16 + 2 * S * 8 + S * sizeof(Job) + kSigRing * 4 + 16;
}

// ---- consumer side ----
// L job: tile of a fused intra-GPU group (alg1 steps 2 + 4 on one GPU, pinned fold, reading R1);
// operand slots 2m / 2m+1 hold x_m / g_m; the mean goes to every member by bulk stores (HBM)
template <bool BF>
__device__ __forceinline__ void consume_L(const XTask& T, const Job& J, const float4* st, float4* out, int ob, int warp,
                                          int lane, int& ncommit) {
  const XLocalGroup& G = T.lg[J.pi];
  const int e0 = warp * kPW;
  const int mine = max(0, min(kPW, J.cnt - e0));
#pragma unroll
  for (int j = 0; j < kVPL; ++j) {
    const int e = e0 + j * 32 + lane;
    if (e >= J.cnt) continue;
    const int64_t i = J.base + e;
    const bool odd_last = BF && (J.cnt & 1) && e == J.cnt - 1;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int m = 0; m < kMaxFusedK; ++m) {
      if (m >= G.k) break;
      float4 x, g, vd;
      if constexpr (BF) {
        if (odd_last) {
          x = unpack_bf4(*reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(G.x[m]) + 4 * i));
          if (G.u[m].g) g = unpack_bf4(*reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(G.u[m].g) + 4 * i));
        } else {
          x = unpack_bf4(reinterpret_cast<const uint2*>(st + (2 * m) * kT)[e]);
          if (G.u[m].g) g = unpack_bf4(reinterpret_cast<const uint2*>(st + (2 * m + 1) * kT)[e]);
        }
      } else {
        x = st[(2 * m) * kT + e];
        if (G.u[m].g) g = st[(2 * m + 1) * kT + e];
      }
      const float4 y = step4<false>(x, g, vd, G.u[m]);
      s = m == 0 ? y : add4(s, y);
    }
    if (G.k > 1) s = div4(s, static_cast<float>(G.k));
    if constexpr (BF) {
      reinterpret_cast<uint2*>(out + ob * kT)[e] = pack_bf4(s);
      if (odd_last)
        for (int m = 0; m < G.k; ++m)
          *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(G.x[m]) + 4 * i) = pack_bf4(s);
    } else {
      out[ob * kT + e] = s;
    }
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0 && mine > 0) {
    int nb = mine;
    if (BF && (J.cnt & 1) && e0 + mine == J.cnt) nb = mine - 1;
    const uint32_t bytes = static_cast<uint32_t>(nb * (BF ? 8 : 16));
    const int64_t off = BF ? 8 * (J.base + e0) : 16 * (J.base + e0);
    const char* srcb = reinterpret_cast<const char*>(BF ? static_cast<const void*>(reinterpret_cast<const uint2*>(out + ob * kT) + e0)
                                                       : static_cast<const void*>(out + ob * kT + e0));
    if (bytes)
      for (int m = 0; m < G.k; ++m) bulk_store(reinterpret_cast<char*>(G.x[m]) + off, srcb, bytes);
  }
  if (lane == 0) {
    bulk_commit();
    ++ncommit;
  }
}

template <bool BF>
__device__ __forceinline__ void tail_L(const XTask& T, int gi, int lane) {
  const XLocalGroup& G = T.lg[gi];
  const int64_t n4 = T.n / 4;
  const int rem = static_cast<int>(T.n - 4 * n4);
  if (lane >= rem) return;
  const int64_t j = 4 * n4 + lane;
  float s = 0.f;
  for (int m = 0; m < G.k; ++m) {
    float y = ldx1<BF>(G.x[m], j);
    if (G.u[m].g) y = step_sgd(y, ldx1<BF>(G.u[m].g, j), G.u[m].lr);
    s = m == 0 ? y : __fadd_rn(s, y);
  }
  if (G.k > 1) s = __fdiv_rn(s, static_cast<float>(G.k));
  for (int m = 0; m < G.k; ++m) stx1<BF>(G.x[m], j, s);
}

template <int M, int KPM, bool BF>
__device__ __forceinline__ void consume(const XTask& T, const Job& J, const float4* st, float4* out, int ob, int warp,
                                        int lane, int& ncommit) {
  const XPart& p = T.part[J.pi];
  const int e0 = warp * kPW;
  const int mine = max(0, min(kPW, J.cnt - e0));
  // operand slot q, vector e: fp32 16 B; bf16 8 B (first half of the slot)
  auto opf = [&](int q, int e) { return st[q * kT + e]; };
  auto opb = [&](int q, int e) { return unpack_bf4(reinterpret_cast<const uint2*>(st + q * kT)[e]); };
  if (J.kind == kJC) {
    // xbar of this tile (slot 0, already rounded for bf16) -> the other local members
#pragma unroll
    for (int j = 0; j < kVPL; ++j) {
      const int e = e0 + j * 32 + lane;
      if (e < J.cnt) {
        if constexpr (BF) reinterpret_cast<uint2*>(out + ob * kT)[e] = reinterpret_cast<const uint2*>(st)[e];
        else out[ob * kT + e] = st[e];
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kVPL; ++j) {
      const int e = e0 + j * 32 + lane;
      if (e >= J.cnt) continue;
      const int64_t i = J.base + e;
      // bf16: an odd last vector of the replica was not bulk-loaded (16-byte granules)
      const bool odd_last = BF && (J.cnt & 1) && e == J.cnt - 1;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        if (m >= p.m) break;
        float4 x, g;
        if constexpr (BF) {
          if (odd_last) {
            const uint2 xw = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(p.x[m]) + 4 * i);
            x = unpack_bf4(xw);
            if (p.u[m].g) g = unpack_bf4(*reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(p.u[m].g) + 4 * i));
          } else {
            x = opb(2 * m, e);
            if (p.u[m].g) g = opb(2 * m + 1, e);
          }
        } else {
          x = opf(2 * m, e);
          if (p.u[m].g) g = opf(2 * m + 1, e);
        }
        float4 vdummy;
        const float4 y = step4<false>(x, g, vdummy, p.u[m]);
        s = m == 0 ? y : add4(s, y);
      }
      if (J.kind == kJA) {
        out[ob * kT + e] = s;  // fp32 partial
      } else {  // B: fold the partials in ascending GPU id, divide (reading R1)
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        int q = 2 * M;
#pragma unroll
        for (int d = 0; d < KPM; ++d) {
          if (d >= p.kp) break;
          const float4 v = d == p.me ? s : opf(q++, e);
          acc = d == 0 ? v : add4(acc, v);
        }
        const float4 xbar = div4(acc, static_cast<float>(p.k_total));
        if constexpr (BF) {
          reinterpret_cast<uint2*>(out + ob * kT)[e] = pack_bf4(xbar);
          if (odd_last) {  // plain stores of the odd last vector (bulk copies move 16-byte granules)
            const uint2 w = pack_bf4(xbar);
            for (int m = 0; m < p.m; ++m) *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.x[m]) + 4 * i) = w;
            for (int d = 0; d < p.kp; ++d)
              if (d != p.me) *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.xfirst[d]) + 4 * i) = w;  // NVLink
          }
        } else {
          out[ob * kT + e] = xbar;
        }
      }
    }
  }
  if (J.kind == kJC && BF && (J.cnt & 1) && lane == 0 && e0 <= J.cnt - 1 && J.cnt - 1 < e0 + kPW) {
    const int64_t i = J.base + J.cnt - 1;  // odd last bf16 vector: not bulk-loaded, copy it directly
    const uint2 w = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(p.x[0]) + 4 * i);
    for (int m = 1; m < p.m; ++m) *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.x[m]) + 4 * i) = w;
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0 && mine > 0) {
    const float4* src = out + ob * kT + e0;
    const char* srcb = reinterpret_cast<const char*>(BF ? static_cast<const void*>(reinterpret_cast<const uint2*>(out + ob * kT) + e0)
                                                       : static_cast<const void*>(src));
    if (J.kind == kJA) {
      const int64_t slo = slice_lo(p, J.o);
      bulk_store(p.stage[J.o] + stage_off(p, p.me, J.base + e0 - slo), src, static_cast<uint32_t>(mine * 16));  // NVLink
    } else {
      int nb = mine;
      if (BF && (J.cnt & 1) && e0 + mine == J.cnt) nb = mine - 1;  // the odd last vector went by plain stores
      const uint32_t bytes = static_cast<uint32_t>(nb * (BF ? 8 : 16));
      const int64_t off = BF ? 8 * (J.base + e0) : 16 * (J.base + e0);
      if (bytes) {
        if (J.kind == kJB) {
          for (int m = 0; m < p.m; ++m) bulk_store(reinterpret_cast<char*>(p.x[m]) + off, srcb, bytes);
          for (int jj = 1; jj < p.kp; ++jj) {
            const int d = (p.me + jj) % p.kp;  // spread the pushes over the peers
            bulk_store(reinterpret_cast<char*>(p.xfirst[d]) + off, srcb, bytes);  // NVLink
          }
        } else {  // C
          for (int m = 1; m < p.m; ++m) bulk_store(reinterpret_cast<char*>(p.x[m]) + off, srcb, bytes);
        }
      }
    }
  }
  if (lane == 0) {
    bulk_commit();
    ++ncommit;
  }
}

// scalar tail of a chunk (warp 0's lanes < rem), after the chunk's last tile job
template <int M, int KPM, bool BF>
__device__ __forceinline__ void tail_job(const XPart& p, int kind, int o, int lane) {
  if (lane >= p.rem) return;
  const int64_t j = 4 * p.n4 + lane;
  if (kind == kJA) {
    const int64_t slo = slice_lo(p, o);
    p.stage[o][stage_off(p, p.me, p.n4 - slo) + lane] = partial1<M, BF>(p, j);  // NVLink (plain store)
  } else if (kind == kJB) {
    const int64_t so = p.n4 - slice_lo(p, p.me);
    const float* stg = p.stage[p.me];
    const float mine = partial1<M, BF>(p, j);
    float s = p.me == 0 ? mine : stg[stage_off(p, 0, so) + lane];
    for (int d = 1; d < p.kp; ++d) s = __fadd_rn(s, d == p.me ? mine : stg[stage_off(p, d, so) + lane]);
    const float xbar = __fdiv_rn(s, static_cast<float>(p.k_total));
    for (int m = 0; m < p.m; ++m) stx1<BF>(p.x[m], j, xbar);
    for (int d = 0; d < p.kp; ++d)
      if (d != p.me) stx1<BF>(p.xfirst[d], j, xbar);  // NVLink
  } else {
    const float v = ldx1<BF>(p.x[0], j);
    for (int m = 1; m < p.m; ++m) stx1<BF>(p.x[m], j, v);
  }
}

// ---- producer side ----
struct Prod {
  int s = 0, it = 0;
  uint32_t phase = 0;
};

template <int NOP, int S>
__device__ __forceinline__ int acquire_stage(Prod& P, uint64_t* empty) {
  if (P.it >= S) mbar_wait(&empty[P.s], P.phase ^ 1u);
  return P.s;
}
template <int S>
__device__ __forceinline__ void advance(Prod& P) {
  ++P.it;
  if (++P.s == S) {
    P.s = 0;
    P.phase ^= 1u;
  }
}

template <int NOP, int S>
__device__ __forceinline__ void produce_marker(int kind, int pi, int64_t pA, int64_t pB, int sig, uint64_t* full,
                                               uint64_t* empty, Job* jobs, Prod& P) {
  const int s = acquire_stage<NOP, S>(P, empty);
  Job& J = jobs[s];
  J.kind = kind;
  J.pi = pi;
  J.cnt = 0;
  J.pA = pA;
  J.pB = pB;
  J.sig = sig;
  J.tail = 0;
  mbar_arrive(&full[s]);
  advance<S>(P);
}

template <int M, int KPM, bool BF, int NOP, int S>
__device__ void produce_tiles(const XTask& T, int pi, int kind, int o, int64_t c, float4* stages, uint64_t* full,
                              uint64_t* empty, Job* jobs, Prod& P, int mk_pi = -1, int64_t mk_pA = -1,
                              int* sig = nullptr) {
  // mk_pA >= 0: a SIG job posting the A flags of (mk_pi, mk_pA) goes in after the first tile
  const XPart& p = T.part[pi];
  bool marked = mk_pA < 0;
  const Range r = chunk_range(p, kind == kJB ? p.me : o, c);
  const bool need_tail = r.tail && (kind != kJC || p.m > 1);
  for (int64_t t0 = r.lo; t0 < r.hi || (t0 == r.lo && need_tail); t0 += kT) {
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kT), r.hi - t0));
    const int s = acquire_stage<NOP, S>(P, empty);
    Job& J = jobs[s];
    J.kind = kind;
    J.pi = pi;
    J.o = o;
    J.cnt = cnt;
    J.base = t0;
    J.tail = need_tail && t0 + kT >= r.hi;
    float4* st = stages + static_cast<size_t>(s) * NOP * kT;
    // bf16 operands: whole 16-byte granules only (an odd last vector is read directly)
    const uint32_t xb = static_cast<uint32_t>(BF ? (cnt & ~1) * 8 : cnt * 16);
    const uint32_t pb = static_cast<uint32_t>(cnt * 16);
    uint32_t tot = 0;
    if (kind == kJC) {
      tot = xb;
    } else {
      for (int m = 0; m < p.m; ++m) tot += p.u[m].g ? 2 * xb : xb;
      if (kind == kJB) tot += (p.kp - 1) * pb;
    }
    if (tot == 0) {
      mbar_arrive(&full[s]);
    } else {
      mbar_expect_tx(&full[s], tot);
      const int64_t eo = BF ? 8 * t0 : 16 * t0;  // byte offset of the tile in a replica
      if (kind == kJC) {
        if (xb) bulk_load(st, reinterpret_cast<const char*>(p.x[0]) + eo, xb, &full[s]);
      } else {
        for (int m = 0; m < p.m; ++m) {
          if (xb) bulk_load(st + (2 * m) * kT, reinterpret_cast<const char*>(p.x[m]) + eo, xb, &full[s]);
          if (p.u[m].g && xb) bulk_load(st + (2 * m + 1) * kT, reinterpret_cast<const char*>(p.u[m].g) + eo, xb, &full[s]);
        }
        if (kind == kJB) {
          const int64_t slo = slice_lo(p, p.me);
          int q = 2 * M;
          for (int d = 0; d < p.kp; ++d)
            if (d != p.me) bulk_load(st + (q++) * kT, p.stage[p.me] + stage_off(p, d, t0 - slo), pb, &full[s]);
        }
      }
    }
    advance<S>(P);
    if (!marked) {
      produce_marker<NOP, S>(kJSig, mk_pi, mk_pA, -1, (*sig)++, full, empty, jobs, P);
      marked = true;
    }
    if (r.hi <= r.lo) break;  // tail-only job
  }
  if (!marked) produce_marker<NOP, S>(kJSig, mk_pi, mk_pA, -1, (*sig)++, full, empty, jobs, P);
}

// L tile q of this launch (group q mod nlocal, tile q / nlocal): x and g of every member
template <bool BF, int NOP, int S>
__device__ void produce_L(const XTask& T, int64_t q, float4* stages, uint64_t* full, uint64_t* empty, Job* jobs,
                          Prod& P) {
  const int64_t n4 = T.n / 4;
  const int64_t tiles = (n4 + kT - 1) / kT;
  const int gi = static_cast<int>(q % T.nlocal);
  const int64_t ti = q / T.nlocal;
  const XLocalGroup& G = T.lg[gi];
  const int64_t t0 = ti * kT;
  const int cnt = static_cast<int>(max(static_cast<int64_t>(0), min(static_cast<int64_t>(kT), n4 - t0)));
  const int s = acquire_stage<NOP, S>(P, empty);
  Job& J = jobs[s];
  J.kind = kJL;
  J.pi = gi;
  J.o = 0;
  J.cnt = cnt;
  J.base = t0;
  J.tail = (ti == max(tiles, static_cast<int64_t>(1)) - 1) && T.n > 4 * n4;
  float4* st = stages + static_cast<size_t>(s) * NOP * kT;
  const uint32_t xb = static_cast<uint32_t>(BF ? (cnt & ~1) * 8 : cnt * 16);
  uint32_t tot = 0;
  for (int m = 0; m < G.k; ++m) tot += G.u[m].g ? 2 * xb : xb;
  if (tot == 0) {
    mbar_arrive(&full[s]);
  } else {
    mbar_expect_tx(&full[s], tot);
    const int64_t eo = BF ? 8 * t0 : 16 * t0;
    for (int m = 0; m < G.k; ++m) {
      bulk_load(st + (2 * m) * kT, reinterpret_cast<const char*>(G.x[m]) + eo, xb, &full[s]);
      if (G.u[m].g) bulk_load(st + (2 * m + 1) * kT, reinterpret_cast<const char*>(G.u[m].g) + eo, xb, &full[s]);
    }
  }
  advance<S>(P);
}


template <int M, int KPM, bool BF, int NOP, int S>
__device__ __forceinline__ void xgpu_ws_body(const XTask& T, int cta, int ncta) {
  extern __shared__ __align__(128) float4 wsmem[];
  float4* stages = wsmem;
  float4* out = stages + static_cast<size_t>(S) * NOP * kT;
  uint64_t* full = reinterpret_cast<uint64_t*>(out + 2 * kT);
  uint64_t* empty = full + S;
  Job* jobs = reinterpret_cast<Job*>(empty + S);
  int* sigcnt = reinterpret_cast<int*>(jobs + S);
  int* abort_w = sigcnt + kSigRing;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    for (int q = 0; q < kSigRing; ++q) sigcnt[q] = 0;
    *abort_w = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int total = T.nparts * kXLanes;
  if (warp == kWarps) {  // ---------------- producer ----------------
    if (lane == 0) {
      if (cta == 0)  // READY: my staging is free for these groups (my previous kernel has finished)
        for (int pi = 0; pi < T.nparts; ++pi) {
          const XPart& p = T.part[pi];
          for (int d = 0; d < p.kp; ++d)
            if (d != p.me) st_release_sys(flag_at(p.pflags[d], p.slot, T.my_gpu, kFlagReady, 0), p.tag[d]);
        }
      Prod P;
      unsigned long long ready_seen = 0;
      int sig = 0;
      bool ok = true;
      // fused intra-GPU groups: this CTA's L tiles q = cta, cta + ncta, ..., spread evenly over
      // its lane iterations (they never wait, so they fill the time flag waits would idle)
      const int64_t ltiles = T.nlocal > 0 ? T.nlocal * max(static_cast<int64_t>(1), (T.n / 4 + kT - 1) / kT) : 0;
      int64_t lq = cta, iters_left = 0;
      for (int idx = cta; idx < total; idx += ncta) {
        const XPart& p = T.part[idx % T.nparts];
        const int ln = idx / T.nparts;
        const int64_t it = ln < p.nch ? (p.nch - 1 - ln) / kXLanes + 1 : 0;
        iters_left += it ? it + 2 * T.blag : 0;
      }
      auto emit_L = [&](bool all) {
        const int64_t left = lq < ltiles ? (ltiles - lq + ncta - 1) / ncta : 0;
        int64_t want = all || iters_left <= 0 ? left : (left + iters_left - 1) / iters_left;
        for (; want > 0 && lq < ltiles; --want, lq += ncta) produce_L<BF, NOP, S>(T, lq, stages, full, empty, jobs, P);
      };
      // ---- one lane iteration's A / B / C blocks (part + chunk each, -1 = none) ----
      auto block_A = [&](int pi, int64_t c) {
        const XPart& p = T.part[pi];
        for (int j = 1; ok && j < p.kp; ++j) {
          const int o = (p.me + j) % p.kp;  // spread the pushes over the owners
          const unsigned long long bit = 1ull << (8 * pi + o);
          if (!(ready_seen & bit)) {
            ok = wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[o], kFlagReady, 0), p.tag[o], p.slot, p.gpu[o],
                           kFlagReady, 0);
            ready_seen |= bit;
          }
          if (ok) produce_tiles<M, KPM, BF, NOP, S>(T, pi, kJA, o, c, stages, full, empty, jobs, P);
        }
      };
      auto block_B = [&](int pi, int64_t c, int mk_pi = -1, int64_t mk_pA = -1) {
        const XPart& p = T.part[pi];
        for (int d = 0; ok && d < p.kp; ++d)
          if (d != p.me)
            ok = wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[d], kFlagA, c), p.tag[d], p.slot, p.gpu[d], kFlagA, c);
        fence_async_all();  // the peers' partials (acquired) are read next by the async proxy
        if (ok) produce_tiles<M, KPM, BF, NOP, S>(T, pi, kJB, p.me, c, stages, full, empty, jobs, P, mk_pi, mk_pA, &sig);
      };
      auto block_C = [&](int pi, int64_t c) {
        const XPart& p = T.part[pi];
        for (int j = 1; ok && j < p.kp; ++j) {
          const int o = (p.me + j) % p.kp;
          ok = wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[o], kFlagB, c), p.tag[o], p.slot, p.gpu[o], kFlagB, c);
          fence_async_all();
          if (ok && p.m > 1) produce_tiles<M, KPM, BF, NOP, S>(T, pi, kJC, o, c, stages, full, empty, jobs, P);
        }
      };
      if (T.claim) {
        // ---- dynamic chunk claiming (default) ----
        // Chunks are claimed from one counter (chunk-major over the parts, parts in ascending seq),
        // so a CTA that runs faster takes more chunks and the kernel has no static tail (the
        // slowest of 296 statically assigned lanes set the kernel time: CTA end times spread
        // 25 % at ResNet-50 size, profiles/r02/). Iteration i: A(claim i), SIG posting B flags of
        // iteration i-1, B(claim i - bl), C(claim i - cl), SIG posting A flags of iteration i.
        // Claims are monotone per GPU in (chunk, group seq), one order shared by all GPUs, and a
        // chunk's A flags depend only on B waits of smaller claims, so no cycle of waits can form.
        constexpr int kRing = 8;
        int cpi[kRing];
        int64_t cch[kRing];
        const int bl = T.blag, cl = T.blag + 1;
        int cur = 0;                   // 1 once the claim counter ran out
        int64_t nclaim = 0;            // claims made by this CTA
        int64_t last = -1;             // iteration of the last successful claim
        int64_t nch_all = 0, max_nch = 0;
        for (int pi = 0; pi < T.nparts; ++pi) {
          nch_all += T.part[pi].nch;
          max_nch = max(max_nch, T.part[pi].nch);
        }
        const int64_t lper = ltiles > 0 ? (ltiles + max(nch_all, static_cast<int64_t>(1)) - 1) / max(nch_all, static_cast<int64_t>(1)) : 0;
        unsigned int* const lctr = T.claim + 2 * kMaxXParts;
        int piB_prev = -1;
        int64_t cB_prev = -1;
        int pre_pi = -1;               // lookahead: a claim whose A block is already pushed
        int64_t pre_c = -1;
        auto claim_next = [&](int& piA, int64_t& cA) {
          // Claim order (the same on every GPU of a group, so no cycle of waits can form):
          // chunk-major (default for Group-Generator steps): every (chunk, part) pair in chunk
          // order, parts ascending seq -- all of a GPU's groups advance together; part-major
          // claiming ran them one after another and chained the GPUs' random groups (-14 % on the
          // 8-worker problem at N = 4). Part-major (static schedules): a GPU in two groups
          // finishes the first early, so that group's peers start their next step while it works
          // on the second -- the fixed schedule turns the skew into overlap across steps
          // (configs[3] layout at N = 4: 5,474 part-major vs 4,430 chunk-major worker-steps/s).
          // profiles/r02/claim_order_4gpu.txt
          while (T.part_major && cur < T.nparts) {  // part-major: a GPU's groups one after another
            const int64_t c = static_cast<int64_t>(atomicAdd(T.claim + 1 + cur, 1u));
            if (c < T.part[cur].nch) {
              piA = cur;
              cA = c;
              break;
            }
            ++cur;
          }
          while (!T.part_major && cur == 0) {
            const int64_t q = static_cast<int64_t>(atomicAdd(T.claim, 1u));
            const int64_t c = q / T.nparts;
            const int pq = static_cast<int>(q - c * T.nparts);
            if (c >= max_nch) {
              cur = 1;  // exhausted
              break;
            }
            if (c < T.part[pq].nch) {
              piA = pq;
              cA = c;
              break;
            }
          }
        };
        // all peers' A flags of (pi, c) posted (non-blocking probe)
        auto a_posted = [&](int pi, int64_t c) {
          const XPart& p = T.part[pi];
          for (int d = 0; d < p.kp; ++d)
            if (d != p.me && ld_acquire_sys(flag_at(T.my_flags, p.slot, p.gpu[d], kFlagA, c)) != p.tag[d]) return false;
          return true;
        };
        for (int64_t i = 0; ok; ++i) {
          int piA = -1;
          int64_t cA = -1;
          bool a_done = false;
          if (pre_c >= 0) {
            piA = pre_pi;
            cA = pre_c;
            pre_c = -1;
            a_done = true;
          } else {
            claim_next(piA, cA);
          }
          if (cA >= 0) {
            cpi[i % kRing] = piA;
            cch[i % kRing] = cA;
            last = i;
            ++nclaim;
          } else if (last < 0 || i > last + cl) {
            break;
          }
          // claims happen in iterations 0 .. last (consecutive, until the counters run out)
          const bool hasB = i - bl >= 0 && i - bl <= last;
          const int piB = hasB ? cpi[(i - bl) % kRing] : -1;
          const int64_t cB = hasB ? cch[(i - bl) % kRing] : -1;
          const bool hasC = i >= cl && i - cl <= last;
          if (cA >= 0 && !a_done) block_A(piA, cA);
          bool sig_a_emitted = false;
          if (ok && piB_prev >= 0) {
            produce_marker<NOP, S>(kJSig, piB_prev, -1, cB_prev, sig++, full, empty, jobs, P);
            piB_prev = -1;
            sig_a_emitted = true;
          }
          // an A block pushed ahead (last iteration, before its B block) is complete once the
          // SIG above has drained (nothing was committed since the last SIG): post its flags now
          if (ok && a_done) produce_marker<NOP, S>(kJSig, piA, cA, -1, sig++, full, empty, jobs, P);
          // early A flags (T.early_a): post this iteration's A flags from a SIG after the first tile of
          // the B block instead of at the iteration's end -- its wait (everything before the SIG above
          // completed) covers the A block, and the peers' B blocks of this claim can start a B block
          // earlier. Needs a SIG between the A block and that one: an empty one if none was posted.
          const bool early = T.early_a && hasB && cA >= 0 && !a_done;
          if (ok && early && !sig_a_emitted) produce_marker<NOP, S>(kJSig, 0, -1, -1, sig++, full, empty, jobs, P);
          if (ok && hasB) {
            // lookahead: the B block's partials are not all in yet -- push the next claim's A
            // block first (it waits for nothing), then block on the flags. Claims stay monotone,
            // and the pushed-ahead A flags are posted at the next iteration's first SIG.
            if (T.lookahead && (T.part_major ? cur < T.nparts : cur == 0) && !a_posted(piB, cB)) {
              claim_next(pre_pi, pre_c);
              if (pre_c >= 0) block_A(pre_pi, pre_c);
            }
            if (ok) {
              if (early) block_B(piB, cB, piA, cA);
              else block_B(piB, cB);
            }
          }
          if (ok && hasC) block_C(cpi[(i - cl) % kRing], cch[(i - cl) % kRing]);
          if (ok) {
            for (int64_t q = 0; q < lper; ++q) {  // fused intra-GPU tiles, claimed as they come
              const int64_t t = static_cast<int64_t>(atomicAdd(lctr, 1u));
              if (t >= ltiles) break;
              produce_L<BF, NOP, S>(T, t, stages, full, empty, jobs, P);
            }
            // always delimit the iteration (even without an A block): the next SIG_a's wait for
            // "only the groups since the last SIG pending" must not cover this iteration's B stores
            produce_marker<NOP, S>(kJSig, cA >= 0 ? piA : 0, a_done || early ? -1 : cA, -1, sig++, full, empty, jobs, P);
          }
          if (hasB) {
            piB_prev = piB;
            cB_prev = cB;
          }
        }
        if (ok && piB_prev >= 0) produce_marker<NOP, S>(kJSig, piB_prev, -1, cB_prev, sig++, full, empty, jobs, P);
        while (ok) {  // leftover fused tiles
          const int64_t t = static_cast<int64_t>(atomicAdd(lctr, 1u));
          if (t >= ltiles) break;
          produce_L<BF, NOP, S>(T, t, stages, full, empty, jobs, P);
        }
        (void)nclaim;
      }
      for (int idx = cta; ok && !T.claim && idx < total; idx += ncta) {
        const int pi = idx % T.nparts, ln = idx / T.nparts;
        const XPart& p = T.part[pi];
        const int64_t iters = ln < p.nch ? (p.nch - 1 - ln) / kXLanes + 1 : 0;
        int64_t pA = -1, pB = -1;
        // B runs bl >= 2 iterations after A (A(c) flags are posted at the end of iteration c+1),
        // C runs 2 bl after A (B(c) flags at the end of iteration c+bl+1)
        // sig2 (default): two SIG jobs per iteration. The one after the A block posts the previous
        // iteration's B flags (its B stores have completed once only the A block's are pending);
        // the one at the end posts this iteration's A flags (only the B / C blocks' pending). A(c)
        // flags then appear at the end of iteration c, so B(c) can run bl >= 1 iteration later,
        // and B(c) flags after the next A block, so C(c) runs cl = bl + 1 iterations after A(c).
        const bool sig2 = T.sig2 != 0;
        const int bl = T.blag, cl = sig2 ? T.blag + 1 : 2 * T.blag;
        for (int64_t i = 0; ok && i < (iters ? iters + cl : 0); ++i) {
          const int64_t cA = i < iters ? ln + i * kXLanes : -1;
          const int64_t cB = (i >= bl && i - bl < iters) ? ln + (i - bl) * kXLanes : -1;
          const int64_t cC = (i >= cl && i - cl < iters) ? ln + (i - cl) * kXLanes : -1;
          if (cA >= 0)
            for (int j = 1; ok && j < p.kp; ++j) {
              const int o = (p.me + j) % p.kp;  // spread the pushes over the owners
              const unsigned long long bit = 1ull << (8 * pi + o);
              if (!(ready_seen & bit)) {
                ok = wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[o], kFlagReady, 0), p.tag[o], p.slot, p.gpu[o],
                               kFlagReady, 0);
                ready_seen |= bit;
              }
              if (ok) produce_tiles<M, KPM, BF, NOP, S>(T, pi, kJA, o, cA, stages, full, empty, jobs, P);
            }
          if (ok && sig2) {
            produce_marker<NOP, S>(kJSig, pi, -1, pB, sig++, full, empty, jobs, P);
            pB = -1;
          }
          if (ok && cB >= 0) {
            for (int d = 0; ok && d < p.kp; ++d)
              if (d != p.me)
                ok = wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[d], kFlagA, cB), p.tag[d], p.slot, p.gpu[d],
                               kFlagA, cB);
            fence_async_all();  // the peers' partials (acquired) are read next by the async proxy
            if (ok) produce_tiles<M, KPM, BF, NOP, S>(T, pi, kJB, p.me, cB, stages, full, empty, jobs, P);
          }
          if (ok && cC >= 0)
            for (int j = 1; ok && j < p.kp; ++j) {
              const int o = (p.me + j) % p.kp;
              ok = wait_flag(T, flag_at(T.my_flags, p.slot, p.gpu[o], kFlagB, cC), p.tag[o], p.slot, p.gpu[o],
                             kFlagB, cC);
              fence_async_all();
              if (ok && p.m > 1) produce_tiles<M, KPM, BF, NOP, S>(T, pi, kJC, o, cC, stages, full, empty, jobs, P);
            }
          if (ok) {
            emit_L(false);
            --iters_left;
            if (sig2)
              produce_marker<NOP, S>(kJSig, pi, cA, -1, sig++, full, empty, jobs, P);
            else
              produce_marker<NOP, S>(kJSig, pi, pA, pB, sig++, full, empty, jobs, P);
          }
          pA = cA;
          pB = cB;
        }
        if (ok && sig2 && pB >= 0)  // the last B block's flags
          produce_marker<NOP, S>(kJSig, pi, -1, pB, sig++, full, empty, jobs, P);
      }
      if (ok && !T.claim) emit_L(true);  // leftovers (and every L tile of a CTA without lane work)
      if (!ok) *reinterpret_cast<volatile int*>(abort_w) = 1;
      produce_marker<NOP, S>(kJEnd, 0, -1, -1, 0, full, empty, jobs, P);
      if (T.claim) {  // the last CTA done claiming resets the counters for the next launch
        __threadfence();
        if (atomicAdd(T.claim + 2 * kMaxXParts + 1, 1u) == static_cast<unsigned>(ncta) - 1) {
          for (int q = 0; q < 2 * kMaxXParts + 1; ++q) T.claim[q] = 0;
          __threadfence();
          T.claim[2 * kMaxXParts + 1] = 0;
        }
      }
    }
    __syncwarp();
  } else {  // ---------------- consumers ----------------
    int ncommit = 0, ntile = 0;
    const unsigned long long t_begin = T.cta_stat && lane == 0 && warp == 0 ? gtimer() : 0;
    for (int it = 0;; ++it) {
      const int s = it % S;
      unsigned long long tw = 0;
      if (T.cta_stat && warp == 0 && lane == 0) tw = gtimer();
      mbar_wait(&full[s], static_cast<uint32_t>((it / S) & 1));
      if (T.cta_stat && warp == 0 && lane == 0) atomicAdd(T.cta_stat + 4 * blockIdx.x + 0, gtimer() - tw);
      const Job J = jobs[s];
      if (J.kind == kJEnd) break;
      if (J.kind == kJSig) {
        if (lane == 0) {
          mbar_arrive(&empty[s]);
          unsigned long long t1 = T.cta_stat && warp == 0 ? gtimer() : 0;
          bulk_wait_pending(ncommit);  // this warp's groups of the previous iteration have completed
          if (T.cta_stat && warp == 0) {
            const unsigned long long t2 = gtimer();
            atomicAdd(T.cta_stat + 4 * blockIdx.x + 1, t2 - t1);
            const unsigned long long q = T.cta_stat[kCtaCntBase + 2 * blockIdx.x]++;
            if (q < kCtaSig)
              T.cta_stat[kCtaSigBase + kCtaSig * blockIdx.x + q] =
                  (t2 & ~3ull) | (J.pA >= 0 ? 1u : 0u) | (J.pB >= 0 ? 2u : 0u);
          }
          ncommit = 0;
          fence_async_all();
          int* cnt = &sigcnt[J.sig % kSigRing];
          if (atom_add_acq_rel_cta(cnt, 1) == kWarps - 1) {  // the last warp posts the flags
            *cnt = 0;
            const XPart& p = T.part[J.pi];
            if (J.pA >= 0 || J.pB >= 0) {
              asm volatile("fence.acq_rel.sys;" ::: "memory");
              if (J.pA >= 0)
                for (int j = 1; j < p.kp; ++j) {
                  const int o = (p.me + j) % p.kp;
                  st_relaxed_sys(flag_at(p.pflags[o], p.slot, T.my_gpu, kFlagA, J.pA), p.tag[o]);
                }
              if (J.pB >= 0)
                for (int d = 0; d < p.kp; ++d)
                  if (d != p.me) st_relaxed_sys(flag_at(p.pflags[d], p.slot, T.my_gpu, kFlagB, J.pB), p.tag[d]);
            }
          }
        }
        __syncwarp();
        continue;
      }
      const float4* st = stages + static_cast<size_t>(s) * NOP * kT;
      // every consumed tile commits one bulk group per warp and alternates the output buffer:
      // the group that read out[ntile & 1] two tiles ago must have finished reading it
      if (lane == 0) bulk_wait_read1();
      __syncwarp();
      if (J.kind == kJL) {
        consume_L<BF>(T, J, st, out, ntile & 1, warp, lane, ncommit);
        ++ntile;
        if (J.tail && warp == 0) tail_L<BF>(T, J.pi, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        continue;
      }
      consume<M, KPM, BF>(T, J, st, out, ntile & 1, warp, lane, ncommit);
      ++ntile;
      // the scalar tail rides on the chunk's last job (warp 0); the other warps release the stage
      if (J.tail && warp == 0) {
        const XPart& p = T.part[J.pi];
        if (J.kind == kJA) tail_job<M, KPM, BF>(p, kJA, J.o, lane);
        else if (J.kind == kJB) tail_job<M, KPM, BF>(p, kJB, 0, lane);
        else tail_job<M, KPM, BF>(p, kJC, J.o, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (lane == 0) bulk_wait_all();
    if (T.cta_stat && warp == 0 && lane == 0) {
      const unsigned long long t_end = gtimer();
      atomicAdd(T.cta_stat + 4 * blockIdx.x + 3, t_end - t_begin);
      T.cta_stat[4 * 2048 + 2 * blockIdx.x] = t_begin;  // absolute begin / end of this CTA's work
      T.cta_stat[4 * 2048 + 2 * blockIdx.x + 1] = t_end;
    }
  }
}

template <int M, int KPM, bool BF, int NOP, int S, int MINB>
__global__ void __launch_bounds__(kWsT, MINB) xgpu_ws_kernel(const __grid_constant__ XTask T) {
  xgpu_ws_body<M, KPM, BF, NOP, S>(T, blockIdx.x, gridDim.x);
}
template <int M, int KPM, bool BF, int NOP, int S, int MINB>
__global__ void __launch_bounds__(kWsT, MINB) xgpu_ws_emul_kernel(const XTask* __restrict__ tasks, int V) {
  const int v = blockIdx.x % V;
  xgpu_ws_body<M, KPM, BF, NOP, S>(tasks[v], blockIdx.x / V, gridDim.x / V);
}

int g_ws_sms = 0;
int ws_sms() {
  if (g_ws_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_ws_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_ws_sms <= 0) g_ws_sms = 148;
  }
  return g_ws_sms;
}

template <int M, int KPM, bool BF, int NOP, int S, int MINB>
int launch_ws_m(XTask& T, const XTask* d_tasks, int V, int max_parts, cudaStream_t stream, std::string* err, bool emu) {
  constexpr size_t smem = ws_smem<NOP, S>();
  static_assert(smem <= 227 * 1024, "shared memory");
  static bool attr = false;
  static int occ = 0, occ_emu = 0;
  if (!attr) {
    if (cudaFuncSetAttribute(xgpu_ws_kernel<M, KPM, BF, NOP, S, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess ||
        cudaFuncSetAttribute(xgpu_ws_emul_kernel<M, KPM, BF, NOP, S, MINB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess) {
      *err = "xgpu_ws: shared memory attribute";
      return RP_ECUDA;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, xgpu_ws_kernel<M, KPM, BF, NOP, S, MINB>, kWsT, smem) !=
            cudaSuccess ||
        occ < 1)
      occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_emu, xgpu_ws_emul_kernel<M, KPM, BF, NOP, S, MINB>, kWsT,
                                                      smem) != cudaSuccess ||
        occ_emu < 1)
      occ_emu = 1;
    attr = true;
  }
  cudaError_t e;
  if (!emu) {
    int64_t grid = static_cast<int64_t>(ws_sms()) * occ;  // every CTA co-resident
    if (T.max_ctas > 0) grid = std::min<int64_t>(grid, T.max_ctas);
    grid = std::max<int64_t>(1, std::min<int64_t>(grid, static_cast<int64_t>(T.nparts) * kXLanes));
    xgpu_ws_kernel<M, KPM, BF, NOP, S, MINB><<<static_cast<int>(grid), kWsT, smem, stream>>>(T);
    e = cudaGetLastError();
  } else {
    const int64_t per =
        std::min<int64_t>(static_cast<int64_t>(ws_sms()) * occ_emu / V, static_cast<int64_t>(max_parts) * kXLanes);
    if (per < 1) {
      *err = "xgpu_ws emulation: more virtual GPUs than resident CTAs";
      return RP_EINVAL;
    }
    auto fn = xgpu_ws_emul_kernel<M, KPM, BF, NOP, S, MINB>;
    void* args[] = {const_cast<XTask**>(&d_tasks), &V};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(static_cast<unsigned>(per * V)),
                                    dim3(kWsT), args, smem, stream);
  }
  if (e != cudaSuccess) {
    *err = std::string("xgpu_ws launch: ") + cudaGetErrorString(e);
    return RP_ECUDA;
  }
  return RP_OK;
}

template <int M, int KPM, bool BF, int NOP, int S, int MINB>
void ws_touch() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, xgpu_ws_kernel<M, KPM, BF, NOP, S, MINB>);
  cudaFuncGetAttributes(&a, xgpu_ws_emul_kernel<M, KPM, BF, NOP, S, MINB>);
}

}  // namespace

// Force-load every instantiation the dispatcher below can pick (CUDA lazy loading would load a
// kernel at its first launch, inside a timed region: 10-11 ms stalls measured in round 2 when a
// random schedule first produced a new (members, GPUs) combination).
void preload_xgpu_ws() {
#define RP_WS(M, KPM, BF, S, MINB) ws_touch<M, KPM, BF, 2 * M + KPM - 1, S, MINB>()
  RP_WS(1, 2, true, 4, 2); RP_WS(1, 2, false, 4, 2); RP_WS(2, 2, true, 2, 2); RP_WS(2, 2, false, 2, 2);
  RP_WS(4, 2, true, 2, 1); RP_WS(4, 2, false, 2, 1); RP_WS(8, 2, true, 1, 1); RP_WS(8, 2, false, 1, 1);
  RP_WS(1, 4, true, 2, 2); RP_WS(1, 4, false, 2, 2); RP_WS(2, 4, true, 3, 1); RP_WS(2, 4, false, 3, 1);
  RP_WS(4, 4, true, 2, 1); RP_WS(4, 4, false, 2, 1); RP_WS(8, 4, true, 1, 1); RP_WS(8, 4, false, 1, 1);
  RP_WS(1, 8, true, 2, 1); RP_WS(1, 8, false, 2, 1); RP_WS(2, 8, true, 2, 1); RP_WS(2, 8, false, 2, 1);
  RP_WS(8, 8, true, 1, 1); RP_WS(8, 8, false, 1, 1);
#undef RP_WS
}

// Operand slots per stage: A needs 2M (x, g of every local member), B 2M + kp - 1 (+ the peers'
// staged partials), C 1. Stages are sized so that two CTAs fit an SM where possible.
int launch_xgpu_ws(XTask& T, const XTask* d_tasks, int V, int max_parts, void* stream, std::string* err, int mmax,
                   int kpmax, bool emu) {
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (T.blag < (T.sig2 ? 1 : 2)) {
    *err = "xgpu_ws: B lag below the flag protocol's minimum";
    return RP_EINVAL;
  }
#define RP_WS(M, KPM, BF, S, MINB) \
  return launch_ws_m<M, KPM, BF, 2 * M + KPM - 1, S, MINB>(T, d_tasks, V, max_parts, s, err, emu)
  const bool bf = T.bf16 != 0;
  (void)emu;  // emulation takes the same instantiation as the real launch
  if (kpmax <= 2) {
    if (mmax <= 1) { if (bf) RP_WS(1, 2, true, 4, 2); RP_WS(1, 2, false, 4, 2); }
    if (mmax <= 2) { if (bf) RP_WS(2, 2, true, 2, 2); RP_WS(2, 2, false, 2, 2); }
    if (mmax <= 4) { if (bf) RP_WS(4, 2, true, 2, 1); RP_WS(4, 2, false, 2, 1); }
    if (bf) RP_WS(8, 2, true, 1, 1);
    RP_WS(8, 2, false, 1, 1);
  }
  if (kpmax <= 4) {
    if (mmax <= 1) { if (bf) RP_WS(1, 4, true, 2, 2); RP_WS(1, 4, false, 2, 2); }
    if (mmax <= 2) { if (bf) RP_WS(2, 4, true, 3, 1); RP_WS(2, 4, false, 3, 1); }
    if (mmax <= 4) { if (bf) RP_WS(4, 4, true, 2, 1); RP_WS(4, 4, false, 2, 1); }
    if (bf) RP_WS(8, 4, true, 1, 1);
    RP_WS(8, 4, false, 1, 1);
  }
  if (mmax <= 1) { if (bf) RP_WS(1, 8, true, 2, 1); RP_WS(1, 8, false, 2, 1); }
  if (mmax <= 2) { if (bf) RP_WS(2, 8, true, 2, 1); RP_WS(2, 8, false, 2, 1); }
  if (bf) RP_WS(8, 8, true, 1, 1);
  RP_WS(8, 8, false, 1, 1);
#undef RP_WS
}

}  // namespace rp
