// Shared helpers for libnekb200 (error state, launch checks, reductions).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cstdarg>
#include <string>
#include <utility>

#include "../../include/nekb200.h"

#define NK_MIN_ORDER 1
#define NK_MAX_ORDER 15
#define NK_GS_MAX_CLASSES 16

namespace nk {

void set_error(const char* fmt, ...);
const char* get_error();

inline cudaStream_t S(nk_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return NK_ERR_CUDA;
  }
  return NK_OK;
}

// Process-wide tuning knobs (nk_set_knob, include/nekb200.h): NK_KNOB_*.
int knob(int k);
// nk_bk5_set_gate: element-count gate of the streamed (chunk-gated) stage BK5
const unsigned long long* bk5_gate();
void set_gate_ptr(const void* p);

// The edge / vertex gather-scatter folded into the tail of the single-rank
// fused BP5 step (nk_bk5_pcg_gs, NK_KNOB_GS_TAIL): the >= 3-member segments
// of a classes plan, one lane per member as in gs_classes_kernel, laid out
// as virtual warps of 32 lanes -- class c owns warps [wstart[c], wstart[c+1]),
// its nseg * Mp lanes padded to a whole warp so no warp mixes classes.
struct GsTail {
  int n;                                  // classes; 0 = no tail
  int M[NK_GS_MAX_CLASSES];               // members per segment
  int Mp[NK_GS_MAX_CLASSES];              // M rounded up to a power of two
  int64_t lanes[NK_GS_MAX_CLASSES];       // nseg * Mp
  const int32_t* mem[NK_GS_MAX_CLASSES];  // member-major local indices
  int64_t wstart[NK_GS_MAX_CLASSES + 1];
};
// host side: nk_bk5_pcg_gs offers its tail to the step launcher for the
// duration of one nk_bk5_pcg call; a launcher that folds it in marks it used
// (anything else leaves it to a separate nk_gs_op_classes launch).
// validate a nk_gs_op_classes class table into a GsTail (T.n = 0: nothing)
int gs_tail_build(GsTail& T, int nclass, const int32_t* sizes, const int64_t* nsegs,
                  const int32_t* const* members);
const GsTail* gs_tail_offer();
void gs_tail_set(const GsTail* t);
void gs_tail_mark_used();
bool gs_tail_used();

// Programmatic dependent launch (PDL).  A kernel launched by launch_ex with
// the knob on may be scheduled while its predecessor in the stream is still
// running; it executes its static-operand prologue (plan indices, G tiles,
// gs codes -- data no kernel writes), then pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible.  Every kernel
// launched through launch_ex calls pdl_wait() on every path before it reads
// or writes anything a predecessor produces, so the relaxation is safe after
// any predecessor (PDL-aware or not).  pdl_trigger() lets the successor
// launch once every CTA of this grid has started.  Both are no-ops for a
// normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// NK_KNOB_PDL bits: which kernel families launch with PDL, and where the
// BP5 step kernel triggers its dependents.
enum {
  kPdlStep = 1,        // fused / split BK5 step (bk5_pencil_tma_pcg, ...)
  kPdlGs = 2,          // gs_classes_kernel
  kPdlVec = 4,         // CG vector kernels (cg_update_gs, cg_xpstep)
  kPdlLateTrigger = 8, // step kernel: trigger after its element loop, not at entry
  kPdlNoPrologue = 16  // step kernel: no G bulk copies before pdl_wait()
};

template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(int family, void (*kern)(KArgs...), dim3 grid, dim3 block,
                             size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (knob(NK_KNOB_PDL) & family) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Fire-and-forget bulk prefetch of [p, p+bytes) into L2 (TMA engine; SASS
// UBLKPF).  Start rounded up and end rounded down to 16 B so the request never
// leaves the allocation.
__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  uintptr_t lo = (a + 15) & ~uintptr_t(15);
  uintptr_t hi = (a + bytes) & ~uintptr_t(15);
  while (lo < hi) {
    const uint32_t n = (uint32_t)((hi - lo) > (1u << 20) ? (1u << 20) : (hi - lo));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(n) : "memory");
    lo += n;
  }
}

// L2 eviction-priority policies (createpolicy; PTX ISA 7.4+) and the
// loads / stores / bulk copies that carry them (.L2::cache_hint).  The BP5
// kernels mark data they stream once per iteration (G, p, x, codes, mask)
// evict_first and the vectors reused across the iteration's kernels (r, w,
// invD) evict_last, so the L2 keeps the reused set while G streams through
// (NK_KNOB_L2).
__device__ __forceinline__ uint64_t l2_policy(int prio) {  // 0 normal, 1 first, 2 last
  uint64_t p;
  if (prio == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (prio == 2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_hint(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_hint(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld2_hint(const double* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ldg2_hint(const double* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ int2 ldg2i_hint(const int32_t* a, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint8_t ldg_u8_hint(const uint8_t* a, uint64_t pol) {
  uint16_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(a), "l"(pol));
  return (uint8_t)v;
}
__device__ __forceinline__ void st_hint(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st2_hint(double* a, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void prefetch_l2_hint(const void* p, int64_t bytes, uint64_t pol) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  uintptr_t lo = (a + 15) & ~uintptr_t(15);
  uintptr_t hi = (a + bytes) & ~uintptr_t(15);
  while (lo < hi) {
    const uint32_t n = (uint32_t)((hi - lo) > (1u << 20) ? (1u << 20) : (hi - lo));
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(lo),
                 "r"(n), "l"(pol)
                 : "memory");
    lo += n;
  }
}
// NK_KNOB_L2 bits
enum { kL2StreamFirst = 1, kL2ReuseLast = 2, kL2InvDLast = 4, kL2SetAside = 8 };
// Host (nk_set_knob(NK_KNOB_L2, ..)): with kL2SetAside, reserve the device's
// maximum persisting-L2 set-aside (cudaLimitPersistingL2CacheSize) for
// evict_last lines; without, release it.
void l2_apply_set_aside();

// Threads per block for the streaming PCG kernels and the fixed number of
// partial sums they produce.  The partial count does not depend on the GPU so
// reductions are bitwise reproducible across devices.
constexpr int kVecThreads = 256;
constexpr int kVecMaxBlocks = 1184;  // 8 x 148 SMs

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sum of NV values per thread; result valid in thread 0.
// `red` must hold NV * 32 doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) red[q * 32 + wid] = v[q];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double t = lane < nw ? red[q * 32 + lane] : 0.0;
      v[q] = warp_sum(t);
    }
  }
  __syncthreads();
}

// Last-block-done: returns true in exactly one block (the last to finish),
// after all other blocks' prior global writes are visible.  Resets the
// ticket so the next launch (or graph replay) starts from zero.
__device__ __forceinline__ bool last_block(uint32_t* ticket, uint32_t nblocks) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t t = atomicAdd(ticket, 1u);
    is_last = (t == nblocks - 1);
    if (is_last) *ticket = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// ---- the edge / vertex gs inside a persistent kernel (nk_bk5_pcg_gs's
// step tail, nk_cg_update_gs's gs prologue) -------------------------------
// The kernel's warps (grid persistent: at most the resident CTA count) work
// through virtual warps gw, gw + nw, ... of the GsTail, kTailU at a time:
// all member-index loads, then all value loads, then per slot the same
// shuffle fold as gs_classes_kernel (member order, ascending local index)
// -- bit-identical to the separate nk_gs_op_classes launch.
constexpr int kTailU = 8;

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// Grid barrier for a grid whose CTAs are all resident: arrival on
// st->ticket[0] (self-resetting, so last_block users of ticket[0] in other
// launches see 0), release through the monotonic st->gen.  Prior global
// writes of every CTA are visible after it.  Returns true in the one CTA
// that arrived last.  Every thread of every CTA must call it.
__device__ __forceinline__ bool grid_barrier(nk_cg_state* st) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t g0 = ld_acquire_u32(&st->gen);
    __threadfence();
    const uint32_t old = atomicAdd(&st->ticket[0], 1u);
    s_last = old == gridDim.x - 1;
    if (s_last) {
      st->ticket[0] = 0u;
      __threadfence();
      atomicAdd(&st->gen, 1u);
    } else {
      while (ld_acquire_u32(&st->gen) == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
  return s_last != 0;
}

__device__ __forceinline__ void gs_tail_idx(const GsTail& T, int64_t v0, int64_t nw, int lane,
                                            int (&idx)[kTailU], int (&cls)[kTailU]) {
  const int64_t W = T.wstart[T.n];
#pragma unroll
  for (int u = 0; u < kTailU; ++u) {
    const int64_t v = v0 + (int64_t)u * nw;
    int c = -1, ix = -1;
    if (v < W) {
      c = 0;
      while (c + 1 < T.n && v >= T.wstart[c + 1]) ++c;
      const int64_t l = (v - T.wstart[c]) * 32 + lane;
      if (l < T.lanes[c]) ix = __ldg(T.mem[c] + l);
    }
    idx[u] = ix;
    cls[u] = c;
  }
}

// w was written by other CTAs of this grid: L2 loads (ld.global.cg), never
// the read-only path
__device__ __forceinline__ void gs_tail_fold(const GsTail& T, double* w, int lane,
                                             const int (&idx)[kTailU], const int (&cls)[kTailU]) {
  double v[kTailU];
#pragma unroll
  for (int u = 0; u < kTailU; ++u) v[u] = idx[u] >= 0 ? __ldcg(w + idx[u]) : 0.0;
#pragma unroll
  for (int u = 0; u < kTailU; ++u) {
    const int c = cls[u];   // warp-uniform
    if (c < 0) continue;
    const int M = T.M[c], Mp = T.Mp[c];
    const int m = lane & (Mp - 1);
    double acc = v[u];
    for (int j = 1; j < M; ++j) acc = acc + __shfl_down_sync(0xffffffffu, v[u], j, Mp);
    const double res = __shfl_sync(0xffffffffu, acc, lane - m);
    if (idx[u] >= 0) w[idx[u]] = res;
  }
}

// Fixed-order sum of partials[0..n) by one block; valid in thread 0.
template <int NV>
__device__ __forceinline__ void reduce_partials(const double* partials, int64_t n,
                                                int64_t stride, double (&out)[NV], double* red) {
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = 0.0;
  // 8 loads in flight per thread, summed in the same (ascending) order as a
  // plain loop -- bit-identical, but the latency of a long partial list (one
  // partial per CTA of a non-persistent BK5 launch: 27648 at N = 3, E = 48^3)
  // is paid once per 8 instead of once per partial.
  constexpr int U = 8;
  int64_t b = threadIdx.x;
  for (; b + (U - 1) * (int64_t)blockDim.x < n; b += U * (int64_t)blockDim.x) {
    double v[U][NV];
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int q = 0; q < NV; ++q) v[k][q] = __ldcg(partials + q * stride + b + k * blockDim.x);
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int q = 0; q < NV; ++q) out[q] += v[k][q];
  }
  for (; b < n; b += blockDim.x) {
#pragma unroll
    for (int q = 0; q < NV; ++q) out[q] += __ldcg(partials + q * stride + b);
  }
  block_sum<NV>(out, red);
}

}  // namespace nk
