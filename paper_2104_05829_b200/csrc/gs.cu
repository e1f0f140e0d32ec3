// Gather-scatter QQ^T on one rank + halo pack/combine (
// PAPER.md:92-141).
//
// The plan is a sorted-index segmented sum: segments in ascending global id,
// members in ascending local index (the canonical order of SPEC.md:205), so a
// sequential fold per segment reproduces the oracle bit-for-bit.  One thread
// per segment; a box mesh has segments of 2 (faces), 4 (edges) and 8
// (vertices).  w is usually still L2-resident from the BK5 launch that wrote
// it, so the random member accesses are served from the 126 MB L2.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace nk {

template <int OP>
__device__ __forceinline__ double fold(double a, double b) {
  if (OP == NK_OP_ADD) return a + b;
  if (OP == NK_OP_MUL) return a * b;
  if (OP == NK_OP_MIN) return fmin(a, b);
  return fmax(a, b);
}
template <int OP>
__device__ __forceinline__ float fold(float a, float b) {   // 32-bit gs
  if (OP == NK_OP_ADD) return a + b;
  if (OP == NK_OP_MUL) return a * b;
  if (OP == NK_OP_MIN) return fminf(a, b);
  return fmaxf(a, b);
}

template <int OP, typename V = double>
__global__ void __launch_bounds__(256)
gs_segments(int64_t nseg, const int32_t* __restrict__ seg_start, const int32_t* __restrict__ perm,
            V* __restrict__ w, int ncomp, int64_t cstride, const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += stride) {
    const int a = __ldg(seg_start + s), b = __ldg(seg_start + s + 1);
    for (int c = 0; c < ncomp; ++c) {
      V* wc = w + c * cstride;
      V acc = wc[__ldg(perm + a)];
      for (int q = a + 1; q < b; ++q) acc = fold<OP>(acc, wc[__ldg(perm + q)]);
      for (int q = a; q < b; ++q) wc[__ldg(perm + q)] = acc;
    }
  }
}

__global__ void gather_kernel(int64_t n, const int32_t* __restrict__ idx,
                              const double* __restrict__ src, double* __restrict__ dst,
                              const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = src[__ldg(idx + i)];
}

template <int OP>
__global__ void halo_combine_kernel(int64_t nh, const int32_t* __restrict__ src_start,
                                    const int32_t* __restrict__ src_idx,
                                    const double* __restrict__ buf,
                                    const int32_t* __restrict__ dst_start,
                                    const int32_t* __restrict__ dst_idx, double* __restrict__ w,
                                    const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += stride) {
    const int a = src_start[h], b = src_start[h + 1];
    double acc = buf[src_idx[a]];
    for (int q = a + 1; q < b; ++q) acc = fold<OP>(acc, buf[src_idx[q]]);
    for (int q = dst_start[h]; q < dst_start[h + 1]; ++q) w[dst_idx[q]] = acc;
  }
}

// Multiplicity classes: the same plan re-packed so every segment of a class
// has M members, stored segment-major and padded to Mp = next power of two
// (<= 32; padding = -1): mem[s * Mp + m].  One LANE per member: each lane
// issues one index load and one value load (a single dependent L2 round
// trip), then the segment's first lane folds the M values, pulled with warp
// shuffles in member order -- the canonical order, so results are
// bit-identical to gs_segments -- and broadcasts the result back.  Segments
// never straddle a warp (Mp divides 32).  Classes with M > 32 use the CSR path.
struct GsClasses {
  int n;
  int M[NK_GS_MAX_CLASSES];
  int Mp[NK_GS_MAX_CLASSES];
  int64_t nseg[NK_GS_MAX_CLASSES];
  const int32_t* mem[NK_GS_MAX_CLASSES];
  int64_t bstart[NK_GS_MAX_CLASSES + 1];
};

// U chunks of 256 lanes per block: each thread issues U independent index
// loads, then U independent value gathers, before any shuffle -- U round
// trips in flight per thread (the kernel is L2-latency-bound, w having just
// been written by BK5).
constexpr int kGsU = 4;

template <int OP, typename V = double>
__global__ void __launch_bounds__(256)
gs_classes_kernel(const __grid_constant__ GsClasses C, V* __restrict__ w, int ncomp,
                  int64_t cs, const nk_cg_state* st) {
  const int64_t b = blockIdx.x;
  int c = 0;
  while (c + 1 < C.n && b >= C.bstart[c + 1]) ++c;
  const int M = C.M[c], Mp = C.Mp[c];
  const int64_t lanes = C.nseg[c] * Mp;
  const int64_t t0 = (b - C.bstart[c]) * (int64_t)(kGsU * blockDim.x) + threadIdx.x;
  // whole warps stay active for the shuffles; out-of-range lanes carry -1.
  // The member indices are plan data (static): loaded before pdl_wait().
  int idx[kGsU];
#pragma unroll
  for (int u = 0; u < kGsU; ++u) {
    const int64_t t = t0 + (int64_t)u * blockDim.x;
    idx[u] = t < lanes ? __ldg(C.mem[c] + t) : -1;
  }
  pdl_wait();
  pdl_trigger();
  if (st != nullptr && st->done) return;
  const int lane = threadIdx.x & 31;
  const int m = lane & (Mp - 1);
  for (int cc = 0; cc < ncomp; ++cc) {
    V* wc = w + cc * cs;
    V v[kGsU];
#pragma unroll
    for (int u = 0; u < kGsU; ++u) v[u] = idx[u] >= 0 ? wc[idx[u]] : V(0);
#pragma unroll
    for (int u = 0; u < kGsU; ++u) {
      V acc = v[u];
      for (int j = 1; j < M; ++j) {
        const V o = __shfl_down_sync(0xffffffffu, v[u], j, Mp);
        acc = fold<OP>(acc, o);
      }
      const V res = __shfl_sync(0xffffffffu, acc, lane - m);
      if (idx[u] >= 0) wc[idx[u]] = res;
    }
  }
}

static unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

int gs_tail_build(GsTail& T, int nclass, const int32_t* sizes, const int64_t* nsegs,
                  const int32_t* const* members) {
  T = GsTail{};
  if (nclass < 0 || nclass > NK_GS_MAX_CLASSES || (nclass > 0 && (!sizes || !nsegs || !members))) {
    set_error("gs classes: invalid class table (max %d classes)", NK_GS_MAX_CLASSES);
    return NK_ERR_INVALID;
  }
  int64_t warps = 0;
  int k = 0;
  for (int c = 0; c < nclass; ++c) {
    if (nsegs[c] <= 0) continue;
    if (sizes[c] < 1 || sizes[c] > 32 || !members[c]) {
      set_error("gs classes: class %d invalid (size %d; 1..32 allowed)", c, sizes[c]);
      return NK_ERR_INVALID;
    }
    int mp = 1;
    while (mp < sizes[c]) mp <<= 1;
    T.M[k] = sizes[c];
    T.Mp[k] = mp;
    T.lanes[k] = nsegs[c] * mp;
    T.mem[k] = members[c];
    T.wstart[k] = warps;
    warps += (T.lanes[k] + 31) / 32;
    ++k;
  }
  T.n = k;
  T.wstart[k] = warps;
  return NK_OK;
}

}  // namespace nk

using namespace nk;

template <typename V>
static int gs_op_t(int64_t nseg, const int32_t* seg_start, const int32_t* perm, V* w, int op,
                   int ncomp, int64_t comp_stride, const nk_cg_state* st, nk_stream_t stream) {
  if (nseg < 0 || (nseg > 0 && (!seg_start || !perm || !w))) {
    set_error("gs_op: invalid plan");
    return NK_ERR_INVALID;
  }
  if (ncomp < 1) {
    set_error("gs_op: ncomp < 1");
    return NK_ERR_INVALID;
  }
  if (nseg == 0) return NK_OK;
  cudaStream_t s = S(stream);
  const unsigned g = grid_for(nseg, 256);
  switch (op) {
    case NK_OP_ADD: gs_segments<NK_OP_ADD, V><<<g, 256, 0, s>>>(nseg, seg_start, perm, w, ncomp, comp_stride, st); break;
    case NK_OP_MUL: gs_segments<NK_OP_MUL, V><<<g, 256, 0, s>>>(nseg, seg_start, perm, w, ncomp, comp_stride, st); break;
    case NK_OP_MIN: gs_segments<NK_OP_MIN, V><<<g, 256, 0, s>>>(nseg, seg_start, perm, w, ncomp, comp_stride, st); break;
    case NK_OP_MAX: gs_segments<NK_OP_MAX, V><<<g, 256, 0, s>>>(nseg, seg_start, perm, w, ncomp, comp_stride, st); break;
    default: set_error("gs_op: unknown op %d", op); return NK_ERR_INVALID;
  }
  return check_launch("gs_segments");
}

extern "C" int nk_gs_op(int64_t nseg, const int32_t* seg_start, const int32_t* perm, double* w,
                        int op, int ncomp, int64_t comp_stride, const nk_cg_state* st,
                        nk_stream_t stream) {
  return gs_op_t<double>(nseg, seg_start, perm, w, op, ncomp, comp_stride, st, stream);
}

extern "C" int nk_gs_op_f32(int64_t nseg, const int32_t* seg_start, const int32_t* perm, float* w,
                            int op, int ncomp, int64_t comp_stride, const nk_cg_state* st,
                            nk_stream_t stream) {
  return gs_op_t<float>(nseg, seg_start, perm, w, op, ncomp, comp_stride, st, stream);
}

template <typename V>
static int gs_op_classes_t(int nclass, const int32_t* sizes, const int64_t* nsegs,
                           const int32_t* const* members, V* w, int op, int ncomp,
                           int64_t comp_stride, const nk_cg_state* st, nk_stream_t stream) {
  if (nclass < 0 || nclass > NK_GS_MAX_CLASSES || (nclass > 0 && (!sizes || !nsegs || !members))) {
    set_error("gs_op_classes: invalid class table (max %d classes)", NK_GS_MAX_CLASSES);
    return NK_ERR_INVALID;
  }
  GsClasses C{};
  int64_t blocks = 0;
  int k = 0;
  for (int c = 0; c < nclass; ++c) {
    if (nsegs[c] <= 0) continue;
    if (sizes[c] < 1 || sizes[c] > 32 || !members[c]) {
      set_error("gs_op_classes: class %d invalid (size %d; 1..32 allowed)", c, sizes[c]);
      return NK_ERR_INVALID;
    }
    int mp = 1;
    while (mp < sizes[c]) mp <<= 1;
    C.M[k] = sizes[c];
    C.Mp[k] = mp;
    C.nseg[k] = nsegs[c];
    C.mem[k] = members[c];
    C.bstart[k] = blocks;
    blocks += (nsegs[c] * mp + 256 * kGsU - 1) / (256 * kGsU);
    ++k;
  }
  C.n = k;
  C.bstart[k] = blocks;
  if (blocks == 0) return NK_OK;
  if (!w) {
    set_error("gs_op_classes: null field");
    return NK_ERR_INVALID;
  }
  cudaStream_t s = S(stream);
  const dim3 g((unsigned)blocks), blk(256);
  switch (op) {
    case NK_OP_ADD: launch_ex(kPdlGs, gs_classes_kernel<NK_OP_ADD, V>, g, blk, 0, s, C, w, ncomp, comp_stride, st); break;
    case NK_OP_MUL: launch_ex(kPdlGs, gs_classes_kernel<NK_OP_MUL, V>, g, blk, 0, s, C, w, ncomp, comp_stride, st); break;
    case NK_OP_MIN: launch_ex(kPdlGs, gs_classes_kernel<NK_OP_MIN, V>, g, blk, 0, s, C, w, ncomp, comp_stride, st); break;
    case NK_OP_MAX: launch_ex(kPdlGs, gs_classes_kernel<NK_OP_MAX, V>, g, blk, 0, s, C, w, ncomp, comp_stride, st); break;
    default: set_error("gs_op_classes: unknown op %d", op); return NK_ERR_INVALID;
  }
  return check_launch("gs_classes");
}

extern "C" int nk_gs_op_classes(int nclass, const int32_t* sizes, const int64_t* nsegs,
                                const int32_t* const* members, double* w, int op, int ncomp,
                                int64_t comp_stride, const nk_cg_state* st, nk_stream_t stream) {
  return gs_op_classes_t<double>(nclass, sizes, nsegs, members, w, op, ncomp, comp_stride, st,
                                 stream);
}

extern "C" int nk_gs_op_classes_f32(int nclass, const int32_t* sizes, const int64_t* nsegs,
                                    const int32_t* const* members, float* w, int op, int ncomp,
                                    int64_t comp_stride, const nk_cg_state* st,
                                    nk_stream_t stream) {
  return gs_op_classes_t<float>(nclass, sizes, nsegs, members, w, op, ncomp, comp_stride, st,
                                stream);
}

extern "C" int nk_gather(int64_t n, const int32_t* idx, const double* src, double* dst,
                         const nk_cg_state* st, nk_stream_t stream) {
  if (n == 0) return NK_OK;
  if (n < 0 || !idx || !src || !dst) {
    set_error("gather: invalid arguments");
    return NK_ERR_INVALID;
  }
  gather_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, idx, src, dst, st);
  return check_launch("gather");
}

extern "C" int nk_halo_combine(int64_t nh, const int32_t* src_start, const int32_t* src_idx,
                               const double* buf, const int32_t* dst_start,
                               const int32_t* dst_idx, double* w, int op,
                               const nk_cg_state* st, nk_stream_t stream) {
  if (nh == 0) return NK_OK;
  if (nh < 0 || !src_start || !src_idx || !buf || !dst_start || !dst_idx || !w) {
    set_error("halo_combine: invalid arguments");
    return NK_ERR_INVALID;
  }
  cudaStream_t s = S(stream);
  const unsigned g = grid_for(nh, 256);
  switch (op) {
    case NK_OP_ADD: halo_combine_kernel<NK_OP_ADD><<<g, 256, 0, s>>>(nh, src_start, src_idx, buf, dst_start, dst_idx, w, st); break;
    case NK_OP_MUL: halo_combine_kernel<NK_OP_MUL><<<g, 256, 0, s>>>(nh, src_start, src_idx, buf, dst_start, dst_idx, w, st); break;
    case NK_OP_MIN: halo_combine_kernel<NK_OP_MIN><<<g, 256, 0, s>>>(nh, src_start, src_idx, buf, dst_start, dst_idx, w, st); break;
    case NK_OP_MAX: halo_combine_kernel<NK_OP_MAX><<<g, 256, 0, s>>>(nh, src_start, src_idx, buf, dst_start, dst_idx, w, st); break;
    default: set_error("halo_combine: unknown op %d", op); return NK_ERR_INVALID;
  }
  return check_launch("halo_combine");
}

// Host: stable counting sort by id (gs_setup for one rank).
extern "C" int nk_gs_plan_build(const int64_t* ids, int64_t n, int32_t* perm, int32_t* seg_start,
                                int64_t* nseg, int64_t* nperm) {
  if (n < 0 || (n > 0 && (!ids || !perm || !seg_start)) || !nseg || !nperm) {
    set_error("gs_plan_build: invalid arguments");
    return NK_ERR_INVALID;
  }
  if (n > INT32_MAX) {
    set_error("gs_plan_build: %lld local points exceed int32 indexing", (long long)n);
    return NK_ERR_INVALID;
  }
  int64_t maxid = 0;
  for (int64_t q = 0; q < n; ++q) maxid = std::max(maxid, ids[q]);
  std::vector<int32_t> cnt((size_t)maxid + 2, 0);
  for (int64_t q = 0; q < n; ++q)
    if (ids[q] > 0) ++cnt[(size_t)ids[q]];
  // offsets of ids with multiplicity >= 2, in ascending id order
  std::vector<int32_t> off((size_t)maxid + 2, -1);
  int64_t np = 0, ns = 0;
  for (int64_t g = 1; g <= maxid; ++g) {
    if (cnt[(size_t)g] >= 2) {
      off[(size_t)g] = (int32_t)np;
      seg_start[ns++] = (int32_t)np;
      np += cnt[(size_t)g];
    }
  }
  seg_start[ns] = (int32_t)np;
  for (int64_t q = 0; q < n; ++q) {  // ascending local index -> stable
    const int64_t g = ids[q];
    if (g > 0 && off[(size_t)g] >= 0) perm[off[(size_t)g]++] = (int32_t)q;
  }
  *nseg = ns;
  *nperm = np;
  return NK_OK;
}

// ------------------------------------------------------------ gs handle
// Library-owned plan (SPEC.md:184-200's GatherScatterHandle for one rank):
// the canonical CSR re-packed by multiplicity class on the device, so a C
// caller needs no host-side re-packing -- nk_gs_create / nk_gs_apply /
// nk_gs_destroy.
struct nk_gs {
  int nclass = 0;
  int32_t sizes[NK_GS_MAX_CLASSES];
  int64_t nsegs[NK_GS_MAX_CLASSES];
  int32_t* mem[NK_GS_MAX_CLASSES];
  int64_t nrest = 0;
  int32_t* rest_seg = nullptr;
  int32_t* rest_idx = nullptr;
  int64_t nseg = 0, nperm = 0;
};

static void gs_free(nk_gs* h) {
  if (!h) return;
  for (int c = 0; c < h->nclass; ++c) cudaFree(h->mem[c]);
  cudaFree(h->rest_seg);
  cudaFree(h->rest_idx);
  delete h;
}

extern "C" int nk_gs_create(const int32_t* perm, const int32_t* seg_start, int64_t nseg,
                            int64_t nperm, nk_gs** out) {
  if (!out || nseg < 0 || nperm < 0 || (nseg > 0 && (!perm || !seg_start))) {
    set_error("gs_create: invalid arguments");
    return NK_ERR_INVALID;
  }
  *out = nullptr;
  nk_gs* h = new nk_gs();
  h->nseg = nseg;
  h->nperm = nperm;
  // classes: distinct segment sizes <= 32, ascending, at most 16; the rest CSR
  std::vector<int> sizes_present;
  for (int64_t s = 0; s < nseg; ++s) {
    const int M = seg_start[s + 1] - seg_start[s];
    if (M >= 1 && M <= 32 &&
        std::find(sizes_present.begin(), sizes_present.end(), M) == sizes_present.end())
      sizes_present.push_back(M);
  }
  std::sort(sizes_present.begin(), sizes_present.end());
  if ((int)sizes_present.size() > NK_GS_MAX_CLASSES) sizes_present.resize(NK_GS_MAX_CLASSES);
  std::vector<int32_t> rest_seg{0}, rest_idx;
  std::vector<std::vector<int32_t>> mems(sizes_present.size());
  for (int64_t s = 0; s < nseg; ++s) {
    const int a = seg_start[s], M = seg_start[s + 1] - a;
    auto it = std::find(sizes_present.begin(), sizes_present.end(), M);
    if (it == sizes_present.end()) {
      for (int m = 0; m < M; ++m) rest_idx.push_back(perm[a + m]);
      rest_seg.push_back((int32_t)rest_idx.size());
      continue;
    }
    const int c = (int)(it - sizes_present.begin());
    int Mp = 1;
    while (Mp < M) Mp <<= 1;
    for (int m = 0; m < Mp; ++m) mems[c].push_back(m < M ? perm[a + m] : -1);
  }
  int rc = NK_OK;
  for (size_t c = 0; c < sizes_present.size() && rc == NK_OK; ++c) {
    int Mp = 1;
    while (Mp < sizes_present[c]) Mp <<= 1;
    h->sizes[c] = sizes_present[c];
    h->nsegs[c] = (int64_t)mems[c].size() / Mp;
    h->mem[c] = nullptr;
    if (cudaMalloc(&h->mem[c], mems[c].size() * sizeof(int32_t)) != cudaSuccess ||
        cudaMemcpy(h->mem[c], mems[c].data(), mems[c].size() * sizeof(int32_t),
                   cudaMemcpyHostToDevice) != cudaSuccess)
      rc = NK_ERR_CUDA;
    h->nclass = (int)c + 1;
  }
  h->nrest = (int64_t)rest_seg.size() - 1;
  if (rc == NK_OK && h->nrest > 0) {
    if (cudaMalloc(&h->rest_seg, rest_seg.size() * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&h->rest_idx, rest_idx.size() * sizeof(int32_t)) != cudaSuccess ||
        cudaMemcpy(h->rest_seg, rest_seg.data(), rest_seg.size() * sizeof(int32_t),
                   cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(h->rest_idx, rest_idx.data(), rest_idx.size() * sizeof(int32_t),
                   cudaMemcpyHostToDevice) != cudaSuccess)
      rc = NK_ERR_CUDA;
  }
  if (rc != NK_OK) {
    set_error("gs_create: device allocation failed: %s", cudaGetErrorString(cudaGetLastError()));
    gs_free(h);
    return rc;
  }
  *out = h;
  return NK_OK;
}

extern "C" int nk_gs_apply(nk_gs* h, double* w, int op, int ncomp, int64_t comp_stride,
                           const nk_cg_state* st, nk_stream_t stream) {
  if (!h) {
    set_error("gs_apply: null handle");
    return NK_ERR_INVALID;
  }
  if (h->nclass > 0) {
    const int32_t* ptrs[NK_GS_MAX_CLASSES];
    for (int c = 0; c < h->nclass; ++c) ptrs[c] = h->mem[c];
    int rc = nk_gs_op_classes(h->nclass, h->sizes, h->nsegs, ptrs, w, op, ncomp, comp_stride,
                              st, stream);
    if (rc != NK_OK) return rc;
  }
  if (h->nrest > 0)
    return nk_gs_op(h->nrest, h->rest_seg, h->rest_idx, w, op, ncomp, comp_stride, st, stream);
  return NK_OK;
}

extern "C" int nk_gs_destroy(nk_gs* h) {
  gs_free(h);
  return NK_OK;
}
