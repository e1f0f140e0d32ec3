// Fused Jacobi-PCG vector kernels.
//
// All scalars (alpha, beta, residual, convergence) stay on the device in an
// nk_cg_state, so an iteration has no host synchronisation and can be
// replayed as a CUDA graph; kernels become no-ops once st->done is set.
// Reductions: each block writes its partial to a fixed slot, and the last
// block to finish sums the slots in index order -- bitwise deterministic
// run to run (no floating-point atomics).  The number of blocks depends only
// on n (vec_grid), never on the device.
#include "common.cuh"

namespace nk {

// NK_KNOB_CG_PIPE applies to vectors up to kPipeMaxN points, whose w / r
// stay largely L2-resident between the BK5 step and the update; above that
// (pure HBM streaming, e.g. configs[2] / [4] on one GPU) the pipelined
// update measured 7% slower (E = 64^3, N = 7: 3.72 vs 3.45 ms per BP5
// iteration, profiles/r2zy_large_n_knobs.jsonl), so large vectors run the
// per-trip form on the 8 x 148-block grid.
constexpr int64_t kPipeMaxN = int64_t(1) << 24;
static int cg_pipe(int64_t n) { return n <= kPipeMaxN ? knob(NK_KNOB_CG_PIPE) : 0; }

// NK_KNOB_CG_PIPE bit 4: cap at 4 x 148 blocks (one resident wave of the
// 64-register update kernels) instead of 8 x 148
static int64_t vec_grid(int64_t n) {
  const int64_t cap = (cg_pipe(n) & 4) ? kVecMaxBlocks / 2 : kVecMaxBlocks;
  int64_t g = (n + kVecThreads - 1) / kVecThreads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return g;
}

__global__ void __launch_bounds__(kVecThreads)
cg_init_kernel(int64_t n, const double* __restrict__ b, double* __restrict__ x,
               double* __restrict__ r, double* __restrict__ p, const double* __restrict__ invD,
               const double* __restrict__ wt, nk_cg_state* st, double* __restrict__ partials,
               double tol, int max_iter, int flexible) {
  __shared__ double red[3 * 32];
  double v[3] = {0.0, 0.0, 0.0};  // bb, rr, rz
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const double bq = b[q];
    const double wq = wt ? wt[q] : 1.0;
    const double zq = invD ? invD[q] * bq : bq;
    x[q] = 0.0;
    r[q] = bq;
    p[q] = zq;
    v[0] = fma(wq * bq, bq, v[0]);
    v[2] = fma(wq * bq, zq, v[2]);
  }
  v[1] = v[0];
  block_sum<3>(v, red);
  const int nb = gridDim.x;
  if (threadIdx.x == 0) {
    partials[0 * kVecMaxBlocks + blockIdx.x] = v[0];
    partials[1 * kVecMaxBlocks + blockIdx.x] = v[1];
    partials[2 * kVecMaxBlocks + blockIdx.x] = v[2];
  }
  if (last_block(&st->ticket[3], nb)) {
    double s[3];
    reduce_partials<3>(partials, nb, kVecMaxBlocks, s, red);
    if (threadIdx.x == 0) {
      st->bb = s[0];
      st->rr = s[1];
      st->rz = s[2];
      st->thresh2 = tol * tol;  // finalize multiplies by the (reduced) bb
      st->max_iter = max_iter;
      st->flexible = flexible ? 1 : 0;
      st->iter = 0;
      st->done = 1;  // armed by nk_cg_init_finalize
    }
  }
}

__global__ void cg_init_finalize_kernel(nk_cg_state* st, double* hist) {
  const double thr = st->thresh2 * st->bb;  // thresh2 holds tol^2 until here
  st->thresh2 = thr;
  st->iter = 0;
  st->converged = 0;
  st->breakdown = 0;
  st->done = 0;
  if (hist) hist[0] = sqrt(st->rr);
  if (st->bb == 0.0 || st->rr <= thr) {
    st->done = 1;
    st->converged = 1;
  }
  if (st->max_iter <= 0) st->done = 1;
}

// Elementwise part of the update for one point; accumulates rr, rz_new, zap.
struct UpdAcc {
  double rr = 0.0, rz = 0.0, zap = 0.0;
};

template <bool FUSED>
__device__ __forceinline__ void upd_point(double alpha, double& x, double& r, double p, double ap,
                                          double invd, double wq, bool has_invd, UpdAcc& a) {
  if (!FUSED) x = fma(alpha, p, x);
  r = fma(-alpha, ap, r);
  const double wr = wq * r;
  a.rr = fma(wr, r, a.rr);
  if (has_invd) {
    const double z = invd * r;
    a.rz = fma(wr, z, a.rz);
    a.zap = fma(wq * z, ap, a.zap);
  }
}

// Assembled value of a point of w and its 1/mult dot weight from the
// per-point gs code (single-rank fused BP5 path, nk_cg_update_gs):
//   code == -1: unshared                        -> Ap = w[q],          wt = 1
//   code >= 0 : 2-member segment, partner index -> Ap = w[q] + w[code], wt = 1/2
//               (a + b == b + a: the bits of the canonical 2-term fold)
//   code <= -2: member of an M = -code segment already assembled in place
//               by the gs over the non-pair segments -> Ap = w[q], wt = 1/M
// rcp: exact 1/m for m < 256 (shared table); larger m divide.
__device__ __forceinline__ void gs_point(int32_t c, double own, double partner, double& ap,
                                         double& wq, const double* rcp) {
  ap = c >= 0 ? own + partner : own;
  wq = c == -1 ? 1.0 : (c >= 0 ? 0.5 : (c > -256 ? rcp[-c] : 1.0 / (double)(-c)));
}

// VEC: 16-byte loads of two consecutive points (all vectors 16-B aligned),
// two pairs in flight per thread per trip for memory-level parallelism.
// FUSED (BP5 fused path): x and p are not touched -- the deferred x update
// and the p update live in bk5_pencil_pcg -- and the iteration counter is
// advanced here.
// GS (implies FUSED): Ap is the pair-unassembled w, assembled per point
// from the gs code (gs_point) -- generic fallback of nk_cg_update_gs.
// Batched (gridDim.y = ncomp components, component c at offset c * cstride
// in r / Ap, state st + c, partials + c * 3 * kVecMaxBlocks): the GS path
// only (nk_cg_update_gs_batch); x / p / invD / wt / code are shared.
template <bool VEC, bool FUSED, bool GS = false>
__global__ void __launch_bounds__(kVecThreads)
cg_update_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                 const double* __restrict__ p, const double* __restrict__ Ap,
                 const double* __restrict__ invD, const double* __restrict__ wt,
                 const uint8_t* __restrict__ mult, nk_cg_state* st,
                 double* __restrict__ partials, const int32_t* __restrict__ code = nullptr,
                 int64_t cstride = 0) {
  __shared__ double red[3 * 32];
  __shared__ double rcp_tab[256];  // exact 1/m for the u8 multiplicity weights
  if (GS && blockIdx.y) {
    r += blockIdx.y * cstride;
    Ap += blockIdx.y * cstride;
    st += blockIdx.y;
    partials += blockIdx.y * 3 * (int64_t)kVecMaxBlocks;
  }
  if (st->done) return;
  if (mult != nullptr || GS) {
    for (int q = threadIdx.x; q < 256; q += blockDim.x) rcp_tab[q] = q ? 1.0 / (double)q : 0.0;
    __syncthreads();
  }
  const double pAp = st->pAp;
  if (!(pAp > 0.0)) {  // indefiniteness / breakdown; uniform branch
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->breakdown = 1;
      st->done = 1;
    }
    return;
  }
  const double alpha = st->rz / pAp;
  const bool hz = invD != nullptr;
  UpdAcc acc;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  auto pair = [&](int64_t q) {
    double2 xv = FUSED ? make_double2(0, 0) : reinterpret_cast<const double2*>(x)[q];
    double2 rv = reinterpret_cast<const double2*>(r)[q];
    const double2 pv = FUSED ? make_double2(0, 0) : __ldg(reinterpret_cast<const double2*>(p) + q);
    double2 av = __ldg(reinterpret_cast<const double2*>(Ap) + q);
    const double2 dv = hz ? __ldg(reinterpret_cast<const double2*>(invD) + q) : make_double2(0, 0);
    double2 wv;
    if (GS) {
      const int2 cv = __ldg(reinterpret_cast<const int2*>(code) + q);
      gs_point(cv.x, av.x, cv.x >= 0 ? Ap[cv.x] : 0.0, av.x, wv.x, rcp_tab);
      gs_point(cv.y, av.y, cv.y >= 0 ? Ap[cv.y] : 0.0, av.y, wv.y, rcp_tab);
    } else if (wt) {
      wv = __ldg(reinterpret_cast<const double2*>(wt) + q);
    } else if (mult) {  // 1-byte multiplicity: the l2 weight is 1/mult
      const uchar2 mv = __ldg(reinterpret_cast<const uchar2*>(mult) + q);
      wv = make_double2(rcp_tab[mv.x], rcp_tab[mv.y]);
    } else {
      wv = make_double2(1, 1);
    }
    upd_point<FUSED>(alpha, xv.x, rv.x, pv.x, av.x, dv.x, wv.x, hz, acc);
    upd_point<FUSED>(alpha, xv.y, rv.y, pv.y, av.y, dv.y, wv.y, hz, acc);
    if (!FUSED) reinterpret_cast<double2*>(x)[q] = xv;
    reinterpret_cast<double2*>(r)[q] = rv;
  };
  if (VEC) {
    const int64_t np = n >> 1;
    int64_t q = gtid;
    for (; q + 3 * nthr < np; q += 4 * nthr) {  // four independent pairs per trip
      pair(q);
      pair(q + nthr);
      pair(q + 2 * nthr);
      pair(q + 3 * nthr);
    }
    for (; q < np; q += nthr) pair(q);
    if ((n & 1) && gtid == 0) {
      const int64_t t = n - 1;
      double xd = 0.0, at = Ap[t], wq = 0.0;
      if (GS) gs_point(code[t], at, code[t] >= 0 ? Ap[code[t]] : 0.0, at, wq, rcp_tab);
      else wq = wt ? wt[t] : (mult ? rcp_tab[mult[t]] : 1.0);
      upd_point<FUSED>(alpha, FUSED ? xd : x[t], r[t], FUSED ? 0.0 : p[t], at,
                       hz ? invD[t] : 0.0, wq, hz, acc);
    }
  } else {
    for (int64_t q = gtid; q < n; q += nthr) {
      double xd = 0.0, aq = Ap[q], wq = 0.0;
      if (GS) gs_point(code[q], aq, code[q] >= 0 ? Ap[code[q]] : 0.0, aq, wq, rcp_tab);
      else wq = wt ? wt[q] : (mult ? rcp_tab[mult[q]] : 1.0);
      upd_point<FUSED>(alpha, FUSED ? xd : x[q], r[q], FUSED ? 0.0 : p[q], aq,
                       hz ? invD[q] : 0.0, wq, hz, acc);
    }
  }
  double v[3] = {acc.rr, acc.rz, acc.zap};
  block_sum<3>(v, red);
  const int nb = gridDim.x;
  if (threadIdx.x == 0) {
    partials[0 * kVecMaxBlocks + blockIdx.x] = v[0];
    partials[1 * kVecMaxBlocks + blockIdx.x] = v[1];
    partials[2 * kVecMaxBlocks + blockIdx.x] = v[2];
  }
  if (last_block(&st->ticket[1], nb)) {
    double s[3];
    reduce_partials<3>(partials, nb, kVecMaxBlocks, s, red);
    if (threadIdx.x == 0) {
      st->rr = s[0];
      if (hz) st->rz_new = s[1];
      st->zap = s[2];
      st->alpha = alpha;
      if (FUSED) st->iter = st->iter + 1;
    }
  }
}

// Gathered segment (code <= -NK_GS_SEG_BASE, nk_cg_update_gs_seg): the point
// belongs to a rank-private segment of M >= 3 members listed at
// tab[k] = M, tab[k+1 .. k+M] = members in canonical order, k = -code -
// NK_GS_SEG_BASE.  Every member folds the whole segment itself, in member
// order -- the canonical fold of gs_classes / gs_segments, so bit-identical
// -- which removes the separate gs pass over edges and vertices.
__device__ __forceinline__ double seg_fold(int32_t c, const double* __restrict__ w,
                                           const int32_t* __restrict__ tab, int& M) {
  const int64_t k = -(int64_t)c - NK_GS_SEG_BASE;
  M = __ldg(tab + k);
  double acc = w[__ldg(tab + k + 1)];
  for (int j = 2; j <= M; ++j) acc += w[__ldg(tab + k + j)];
  return acc;
}

// gs_point plus the gathered-segment code: pv = the partner value or the
// segment fold, m = M for a gathered segment.
__device__ __forceinline__ void gs_point_seg(int32_t c, double own, double pv, int m, double& ap,
                                             double& wq, const double* rcp) {
  if (c <= -NK_GS_SEG_BASE) {
    ap = pv;
    wq = m < 256 ? rcp[m] : 1.0 / (double)m;
  } else {
    gs_point(c, own, pv, ap, wq, rcp);
  }
}

// nk_cg_update_gs, 16-B path: the cg_update_kernel<true, true, true> loop
// restructured so that every load of a trip is issued before any is used
// -- codes, r, w, invD of a pair, then the pair partners (or, SEG, the
// gathered segments) -- instead of a dependent chain per point; same
// per-thread point order and accumulation as the generic form
// (bit-identical sums).
// PDL prologue: the reciprocal table and the first trip's code / invD
// (static operands) are loaded before pdl_wait().
// pf > 0 (NK_KNOB_CG_UPDATE): the block's contiguous 256-pair segment of
// trip k + pf (r, w, invD, code) is bulk-prefetched into L2 by thread 0
// during trip k, so each trip's loads are L2 hits and HBM streams
// continuously.
// Batched like cg_update_kernel: gridDim.y components at cstride.
// PIPE (NK_KNOB_CG_PIPE): software-pipelined across trips -- trip k + 1's
// code / invD / r / w are loaded into registers while trip k's partner
// gather and update run, so a trip waits on ONE dependent load (the
// partner, whose code is already in a register) instead of code -> partner.
// Same per-thread point order and accumulation (bit-identical).
// PIPE2: two deep -- the code runs two trips ahead and the partner load
// one trip ahead, so no load of a trip is issued in the trip that uses it.
template <bool SEG, int PIPE = 0>
__global__ void __launch_bounds__(kVecThreads, 4)
cg_update_gs_vec_kernel(int64_t n, double* __restrict__ r, const double* __restrict__ w,
                        const double* __restrict__ invD, const int32_t* __restrict__ code,
                        const int32_t* __restrict__ tab, nk_cg_state* st,
                        double* __restrict__ partials, int64_t cstride, int pf,
                        int l2_flags) {
  __shared__ double red[3 * 32];
  __shared__ double rcp_tab[256];
  for (int q = threadIdx.x; q < 256; q += blockDim.x) rcp_tab[q] = q ? 1.0 / (double)q : 0.0;
  const bool hz = invD != nullptr;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t np = n >> 1;
  const uint64_t pol_s = l2_policy(l2_flags & kL2StreamFirst ? 1 : 0);   // code
  const uint64_t pol_r = l2_policy(l2_flags & kL2ReuseLast ? 2 : 0);     // r, w
  const uint64_t pol_d = l2_policy(l2_flags & kL2InvDLast ? 2 : 0);      // invD
  // bulk L2 prefetch of trip k's block segment: static arrays, or r / w
  auto pf_trip = [&](int64_t k, bool stat, bool dyn) {
    const int64_t q0 = k * nthr + (int64_t)blockIdx.x * blockDim.x;
    if (q0 >= np) return;
    const int64_t cnt = np - q0 < (int64_t)blockDim.x ? np - q0 : (int64_t)blockDim.x;
    if (stat) {
      prefetch_l2_hint(code + 2 * q0, cnt * 8, pol_s);
      if (hz) prefetch_l2_hint(invD + 2 * q0, cnt * 16, pol_d);
    }
    if (dyn) {
      prefetch_l2_hint(r + 2 * q0, cnt * 16, pol_r);  // r, w: offset to component blockIdx.y
      prefetch_l2_hint(w + 2 * q0, cnt * 16, pol_r);
    }
  };
  if (threadIdx.x == 0)
    for (int k = 1; k <= pf; ++k) pf_trip(k, true, false);
  int2 cv = gtid < np ? ldg2i_hint(code + 2 * gtid, pol_s) : make_int2(-1, -1);
  double2 dv = (gtid < np && hz) ? ldg2_hint(invD + 2 * gtid, pol_d) : make_double2(0, 0);
  pdl_wait();
  pdl_trigger();
  if (blockIdx.y) {
    r += blockIdx.y * cstride;
    w += blockIdx.y * cstride;
    st += blockIdx.y;
    partials += blockIdx.y * 3 * (int64_t)kVecMaxBlocks;
  }
  if (st->done) return;
  __syncthreads();
  const double pAp = st->pAp;
  if (!(pAp > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->breakdown = 1;
      st->done = 1;
    }
    return;
  }
  const double alpha = st->rz / pAp;
  UpdAcc acc;
  auto gather = [&](int32_t c, int& m) -> double {
    m = 0;
    if (c >= 0) return w[c];
    if (SEG && c <= -NK_GS_SEG_BASE) return seg_fold(c, w, tab, m);
    return 0.0;
  };
  if (threadIdx.x == 0)
    for (int k = 1; k <= pf; ++k) pf_trip(k, false, true);
  int64_t k = 0;
  if constexpr (PIPE == 2) {
    static_assert(!SEG, "two-deep pipeline: pair / unshared codes only");
    double2 rv = make_double2(0, 0), av = make_double2(0, 0);
    double px = 0.0, py = 0.0;
    int2 cv1 = make_int2(-1, -1);
    if (gtid < np) {
      rv = ld2_hint(r + 2 * gtid, pol_r);
      av = ldg2_hint(w + 2 * gtid, pol_r);
      if (cv.x >= 0) px = w[cv.x];
      if (cv.y >= 0) py = w[cv.y];
      if (gtid + nthr < np) cv1 = ldg2i_hint(code + 2 * (gtid + nthr), pol_s);
    }
    for (int64_t q = gtid; q < np; q += nthr, ++k) {
      if (pf > 0 && threadIdx.x == 0) pf_trip(k + 1 + pf, true, true);
      const int64_t qn = q + nthr;
      double2 dvn = make_double2(0, 0), rvn = make_double2(0, 0), avn = make_double2(0, 0);
      double pxn = 0.0, pyn = 0.0;
      int2 cv2 = make_int2(-1, -1);
      if (qn < np) {
        if (hz) dvn = ldg2_hint(invD + 2 * qn, pol_d);
        rvn = ld2_hint(r + 2 * qn, pol_r);
        avn = ldg2_hint(w + 2 * qn, pol_r);
        if (cv1.x >= 0) pxn = w[cv1.x];
        if (cv1.y >= 0) pyn = w[cv1.y];
        if (qn + nthr < np) cv2 = ldg2i_hint(code + 2 * (qn + nthr), pol_s);
      }
      double2 wv;
      gs_point_seg(cv.x, av.x, px, 0, av.x, wv.x, rcp_tab);
      gs_point_seg(cv.y, av.y, py, 0, av.y, wv.y, rcp_tab);
      double xd = 0.0;
      upd_point<true>(alpha, xd, rv.x, 0.0, av.x, dv.x, wv.x, hz, acc);
      upd_point<true>(alpha, xd, rv.y, 0.0, av.y, dv.y, wv.y, hz, acc);
      st2_hint(r + 2 * q, rv, pol_r);
      cv = cv1;
      cv1 = cv2;
      dv = dvn;
      rv = rvn;
      av = avn;
      px = pxn;
      py = pyn;
    }
  } else if constexpr (PIPE == 1) {
    double2 rv = make_double2(0, 0), av = make_double2(0, 0);
    if (gtid < np) {
      rv = ld2_hint(r + 2 * gtid, pol_r);
      av = ldg2_hint(w + 2 * gtid, pol_r);
    }
    for (int64_t q = gtid; q < np; q += nthr, ++k) {
      if (pf > 0 && threadIdx.x == 0) pf_trip(k + 1 + pf, true, true);
      int mx, my;
      const double px = gather(cv.x, mx), py = gather(cv.y, my);
      const int64_t qn = q + nthr;
      int2 cvn = make_int2(-1, -1);
      double2 dvn = make_double2(0, 0), rvn = make_double2(0, 0), avn = make_double2(0, 0);
      if (qn < np) {
        cvn = ldg2i_hint(code + 2 * qn, pol_s);
        if (hz) dvn = ldg2_hint(invD + 2 * qn, pol_d);
        rvn = ld2_hint(r + 2 * qn, pol_r);
        avn = ldg2_hint(w + 2 * qn, pol_r);
      }
      double2 wv;
      gs_point_seg(cv.x, av.x, px, mx, av.x, wv.x, rcp_tab);
      gs_point_seg(cv.y, av.y, py, my, av.y, wv.y, rcp_tab);
      double xd = 0.0;
      upd_point<true>(alpha, xd, rv.x, 0.0, av.x, dv.x, wv.x, hz, acc);
      upd_point<true>(alpha, xd, rv.y, 0.0, av.y, dv.y, wv.y, hz, acc);
      st2_hint(r + 2 * q, rv, pol_r);
      cv = cvn;
      dv = dvn;
      rv = rvn;
      av = avn;
    }
  } else
  for (int64_t q = gtid; q < np; q += nthr, ++k) {
    if (pf > 0 && threadIdx.x == 0) pf_trip(k + 1 + pf, true, true);
    if (q != gtid) {
      cv = ldg2i_hint(code + 2 * q, pol_s);
      dv = hz ? ldg2_hint(invD + 2 * q, pol_d) : make_double2(0, 0);
    }
    double2 rv = ld2_hint(r + 2 * q, pol_r);
    double2 av = ldg2_hint(w + 2 * q, pol_r);
    int mx, my;
    const double px = gather(cv.x, mx), py = gather(cv.y, my);
    double2 wv;
    gs_point_seg(cv.x, av.x, px, mx, av.x, wv.x, rcp_tab);
    gs_point_seg(cv.y, av.y, py, my, av.y, wv.y, rcp_tab);
    double xd = 0.0;
    upd_point<true>(alpha, xd, rv.x, 0.0, av.x, dv.x, wv.x, hz, acc);
    upd_point<true>(alpha, xd, rv.y, 0.0, av.y, dv.y, wv.y, hz, acc);
    st2_hint(r + 2 * q, rv, pol_r);
  }
  if ((n & 1) && gtid == 0) {
    const int64_t t = n - 1;
    double xd = 0.0, at = 0.0, wq = 0.0;
    int m;
    const double pt = gather(code[t], m);
    gs_point_seg(code[t], w[t], pt, m, at, wq, rcp_tab);
    upd_point<true>(alpha, xd, r[t], 0.0, at, hz ? invD[t] : 0.0, wq, hz, acc);
  }
  double v[3] = {acc.rr, acc.rz, acc.zap};
  block_sum<3>(v, red);
  const int nb = gridDim.x;
  if (threadIdx.x == 0) {
    partials[0 * kVecMaxBlocks + blockIdx.x] = v[0];
    partials[1 * kVecMaxBlocks + blockIdx.x] = v[1];
    partials[2 * kVecMaxBlocks + blockIdx.x] = v[2];
  }
  if (last_block(&st->ticket[1], nb)) {
    double sres[3];
    reduce_partials<3>(partials, nb, kVecMaxBlocks, sres, red);
    if (threadIdx.x == 0) {
      st->rr = sres[0];
      if (hz) st->rz_new = sres[1];
      st->zap = sres[2];
      st->alpha = alpha;
      st->iter = st->iter + 1;
    }
  }
}

template <bool VEC>
__global__ void __launch_bounds__(kVecThreads)
cg_pupdate_kernel(int64_t n, const double* __restrict__ r, double* __restrict__ p,
                  const double* __restrict__ invD, const double* __restrict__ z, nk_cg_state* st,
                  double* __restrict__ hist) {
  if (st->done) return;
  const bool conv = st->rr <= st->thresh2;
  const double rz = st->rz;
  const double beta = st->flexible ? (-st->alpha * st->zap) / rz : st->rz_new / rz;
  if (!conv) {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    if (VEC) {
      const int64_t np = n >> 1;
#pragma unroll 2
      for (int64_t q = gtid; q < np; q += nthr) {
        double2 zv;
        if (z) {
          zv = __ldg(reinterpret_cast<const double2*>(z) + q);
        } else {
          const double2 rv = __ldg(reinterpret_cast<const double2*>(r) + q);
          const double2 dv = invD ? __ldg(reinterpret_cast<const double2*>(invD) + q)
                                  : make_double2(1.0, 1.0);
          zv = make_double2(dv.x * rv.x, dv.y * rv.y);
        }
        double2 pv = reinterpret_cast<const double2*>(p)[q];
        pv.x = fma(beta, pv.x, zv.x);
        pv.y = fma(beta, pv.y, zv.y);
        reinterpret_cast<double2*>(p)[q] = pv;
      }
      if ((n & 1) && gtid == 0) {
        const int64_t q = n - 1;
        const double zq = z ? z[q] : (invD ? invD[q] * r[q] : r[q]);
        p[q] = fma(beta, p[q], zq);
      }
    } else {
      for (int64_t q = gtid; q < n; q += nthr) {
        const double zq = z ? z[q] : (invD ? invD[q] * r[q] : r[q]);
        p[q] = fma(beta, p[q], zq);
      }
    }
  }
  if (last_block(&st->ticket[2], gridDim.x)) {
    if (threadIdx.x == 0) {
      const int it = st->iter + 1;
      st->iter = it;
      if (hist) hist[it] = sqrt(st->rr);
      if (conv) {
        st->converged = 1;
        st->done = 1;
      } else {
        st->rz = st->rz_new;
        if (it >= st->max_iter) st->done = 1;
      }
    }
  }
}

__global__ void __launch_bounds__(kVecThreads)
wdot_partial_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                    const double* __restrict__ wt, double* __restrict__ partials) {
  __shared__ double red[32];
  double v[1] = {0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const double t = a[q] * b[q];
    v[0] = wt ? fma(wt[q], t, v[0]) : v[0] + t;
  }
  block_sum<1>(v, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
}

__global__ void __launch_bounds__(kVecThreads)
wdot_final_kernel(int64_t nb, const double* __restrict__ partials, double* out) {
  __shared__ double red[32];
  double s[1];
  reduce_partials<1>(partials, nb, 0, s, red);
  if (threadIdx.x == 0) out[0] = s[0];
}

}  // namespace nk

using namespace nk;

template <typename... T>
static bool aligned16(const T*... ptrs) {
  bool ok = true;
  ((ok = ok && (reinterpret_cast<uintptr_t>(ptrs) & 15) == 0), ...);
  return ok;
}

extern "C" int64_t nk_cg_partials_len(int64_t n) { return 3 * (int64_t)kVecMaxBlocks; }

extern "C" int nk_cg_init(int64_t n, const double* b, double* x, double* r, double* p,
                          const double* invD, const double* wt, nk_cg_state* st,
                          double* partials, double tol, int max_iter, int flexible,
                          nk_stream_t stream) {
  if (n < 0 || !b || !x || !r || !p || !st || !partials) {
    set_error("cg_init: invalid arguments");
    return NK_ERR_INVALID;
  }
  cudaStream_t s = S(stream);
  cg_init_kernel<<<(unsigned)vec_grid(n), kVecThreads, 0, s>>>(n, b, x, r, p, invD, wt, st,
                                                               partials, tol, max_iter, flexible);
  return check_launch("cg_init");
}

extern "C" int nk_cg_init_finalize(nk_cg_state* st, double* hist, nk_stream_t stream) {
  if (!st) {
    set_error("cg_init_finalize: null state");
    return NK_ERR_INVALID;
  }
  cg_init_finalize_kernel<<<1, 1, 0, S(stream)>>>(st, hist);
  return check_launch("cg_init_finalize");
}

extern "C" int nk_cg_update(int64_t n, double* x, double* r, const double* p, const double* Ap,
                            const double* invD, const double* wt, const uint8_t* mult,
                            nk_cg_state* st, double* partials, nk_stream_t stream) {
  if (n < 0 || !r || !Ap || !st || !partials || (x != nullptr && p == nullptr)) {
    set_error("cg_update: invalid arguments");
    return NK_ERR_INVALID;
  }
  const unsigned g = (unsigned)vec_grid(n);
  cudaStream_t s = S(stream);
  const bool vec = aligned16(x, r, p, Ap, invD, wt) && (((uintptr_t)mult & 1) == 0);
  if (x == nullptr) {  // fused BP5 path
    if (vec)
      cg_update_kernel<true, true><<<g, kVecThreads, 0, s>>>(n, x, r, p, Ap, invD, wt, mult, st, partials);
    else
      cg_update_kernel<false, true><<<g, kVecThreads, 0, s>>>(n, x, r, p, Ap, invD, wt, mult, st, partials);
  } else if (vec) {
    cg_update_kernel<true, false><<<g, kVecThreads, 0, s>>>(n, x, r, p, Ap, invD, wt, mult, st, partials);
  } else {
    cg_update_kernel<false, false><<<g, kVecThreads, 0, s>>>(n, x, r, p, Ap, invD, wt, mult, st, partials);
  }
  return check_launch("cg_update");
}

extern "C" int nk_cg_update_gs_seg(int64_t n, int ncomp, int64_t cstride, double* r,
                                   const double* w, const double* invD, const int32_t* code,
                                   const int32_t* segtab, nk_cg_state* st, double* partials,
                                   nk_stream_t stream) {
  if (n < 0 || ncomp < 1 || ncomp > 65535 || (ncomp > 1 && cstride < n) || !r || !w || !code ||
      !st || !partials) {
    set_error("cg_update_gs: invalid arguments");
    return NK_ERR_INVALID;
  }
  const dim3 g((unsigned)vec_grid(n), (unsigned)ncomp);
  cudaStream_t s = S(stream);
  if (aligned16(r, w, invD) && ((uintptr_t)code & 7) == 0 && (cstride % 2 == 0 || ncomp == 1)) {
    const int pf = knob(NK_KNOB_CG_UPDATE);
    if (segtab)
      launch_ex(kPdlVec, cg_update_gs_vec_kernel<true>, g, dim3(kVecThreads), 0, s, n, r, w,
                invD, code, segtab, st, partials, cstride, pf, knob(NK_KNOB_L2));
    else if ((cg_pipe(n) & 3) == 2)
      launch_ex(kPdlVec, cg_update_gs_vec_kernel<false, 2>, g, dim3(kVecThreads), 0, s, n, r,
                w, invD, code, segtab, st, partials, cstride, pf, knob(NK_KNOB_L2));
    else if ((cg_pipe(n) & 3) == 1)
      launch_ex(kPdlVec, cg_update_gs_vec_kernel<false, 1>, g, dim3(kVecThreads), 0, s, n, r,
                w, invD, code, segtab, st, partials, cstride, pf, knob(NK_KNOB_L2));
    else
      launch_ex(kPdlVec, cg_update_gs_vec_kernel<false>, g, dim3(kVecThreads), 0, s, n, r, w,
                invD, code, segtab, st, partials, cstride, pf, knob(NK_KNOB_L2));
  } else {
    if (segtab) {
      set_error("cg_update_gs_seg: gathered segments need 16-byte aligned r / w / invD");
      return NK_ERR_INVALID;
    }
    cg_update_kernel<false, true, true><<<g, kVecThreads, 0, s>>>(
        n, nullptr, r, nullptr, w, invD, nullptr, nullptr, st, partials, code, cstride);
  }
  return check_launch("cg_update_gs");
}

extern "C" int nk_cg_update_gs_batch(int64_t n, int ncomp, int64_t cstride, double* r,
                                     const double* w, const double* invD, const int32_t* code,
                                     nk_cg_state* st, double* partials, nk_stream_t stream) {
  return nk_cg_update_gs_seg(n, ncomp, cstride, r, w, invD, code, nullptr, st, partials, stream);
}

extern "C" int nk_cg_update_gs(int64_t n, double* r, const double* w, const double* invD,
                               const int32_t* code, nk_cg_state* st, double* partials,
                               nk_stream_t stream) {
  return nk_cg_update_gs_batch(n, 1, 0, r, w, invD, code, st, partials, stream);
}

// nk_cg_update_gs_cls, NK_KNOB_GS_TAIL = 2: the gs over the >= 3-member
// segments run by the update kernel itself before its first trip (one launch
// instead of gs_classes_kernel + cg_update_gs_vec_kernel<false, 2>).  The
// grid is one resident wave (vec_grid: 4 x 148 blocks of 256 threads), so
// after its share of the segments every CTA meets a grid barrier, then runs
// the two-deep pipelined update of cg_update_gs_vec_kernel<false, 2> (same
// per-thread point order and accumulation: bit-identical) with w read through
// coherent (non-.nc) loads, since this launch wrote it.
__global__ void __launch_bounds__(kVecThreads, 4)
cg_update_gs_pre_kernel(int64_t n, double* __restrict__ r, double* w,
                        const double* __restrict__ invD, const int32_t* __restrict__ code,
                        nk_cg_state* st, double* __restrict__ partials,
                        const __grid_constant__ GsTail tail, int pf, int l2_flags) {
  __shared__ double red[3 * 32];
  __shared__ double rcp_tab[256];
  for (int q = threadIdx.x; q < 256; q += blockDim.x) rcp_tab[q] = q ? 1.0 / (double)q : 0.0;
  const bool hz = invD != nullptr;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t np = n >> 1;
  const uint64_t pol_s = l2_policy(l2_flags & kL2StreamFirst ? 1 : 0);   // code
  const uint64_t pol_r = l2_policy(l2_flags & kL2ReuseLast ? 2 : 0);     // r, w
  const uint64_t pol_d = l2_policy(l2_flags & kL2InvDLast ? 2 : 0);      // invD
  auto pf_trip = [&](int64_t k, bool stat, bool dyn) {
    const int64_t q0 = k * nthr + (int64_t)blockIdx.x * blockDim.x;
    if (q0 >= np) return;
    const int64_t cnt = np - q0 < (int64_t)blockDim.x ? np - q0 : (int64_t)blockDim.x;
    if (stat) {
      prefetch_l2_hint(code + 2 * q0, cnt * 8, pol_s);
      if (hz) prefetch_l2_hint(invD + 2 * q0, cnt * 16, pol_d);
    }
    if (dyn) {
      prefetch_l2_hint(r + 2 * q0, cnt * 16, pol_r);
      prefetch_l2_hint(w + 2 * q0, cnt * 16, pol_r);
    }
  };
  if (threadIdx.x == 0)
    for (int k = 1; k <= pf; ++k) pf_trip(k, true, false);
  int2 cv = gtid < np ? ldg2i_hint(code + 2 * gtid, pol_s) : make_int2(-1, -1);
  double2 dv = (gtid < np && hz) ? ldg2_hint(invD + 2 * gtid, pol_d) : make_double2(0, 0);
  // the gs plan is static: the first round's member indices before pdl_wait
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t W = tail.wstart[tail.n];
  int idx[kTailU], cls[kTailU];
  gs_tail_idx(tail, gw, nw, lane, idx, cls);
  pdl_wait();
  pdl_trigger();
  if (st->done) return;               // uniform over the grid: before the barrier
  __syncthreads();
  const double pAp = st->pAp;
  if (!(pAp > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->breakdown = 1;
      st->done = 1;
    }
    return;
  }
  const double alpha = st->rz / pAp;
  for (int64_t v0 = gw; v0 < W; v0 += (int64_t)kTailU * nw) {
    if (v0 != gw) gs_tail_idx(tail, v0, nw, lane, idx, cls);
    gs_tail_fold(tail, w, lane, idx, cls);
  }
  grid_barrier(st);
  UpdAcc acc;
  if (threadIdx.x == 0)
    for (int k = 1; k <= pf; ++k) pf_trip(k, false, true);
  int64_t k = 0;
  double2 rv = make_double2(0, 0), av = make_double2(0, 0);
  double px = 0.0, py = 0.0;
  int2 cv1 = make_int2(-1, -1);
  if (gtid < np) {
    rv = ld2_hint(r + 2 * gtid, pol_r);
    av = ld2_hint(w + 2 * gtid, pol_r);
    if (cv.x >= 0) px = __ldcg(w + cv.x);
    if (cv.y >= 0) py = __ldcg(w + cv.y);
    if (gtid + nthr < np) cv1 = ldg2i_hint(code + 2 * (gtid + nthr), pol_s);
  }
  for (int64_t q = gtid; q < np; q += nthr, ++k) {
    if (pf > 0 && threadIdx.x == 0) pf_trip(k + 1 + pf, true, true);
    const int64_t qn = q + nthr;
    double2 dvn = make_double2(0, 0), rvn = make_double2(0, 0), avn = make_double2(0, 0);
    double pxn = 0.0, pyn = 0.0;
    int2 cv2 = make_int2(-1, -1);
    if (qn < np) {
      if (hz) dvn = ldg2_hint(invD + 2 * qn, pol_d);
      rvn = ld2_hint(r + 2 * qn, pol_r);
      avn = ld2_hint(w + 2 * qn, pol_r);
      if (cv1.x >= 0) pxn = __ldcg(w + cv1.x);
      if (cv1.y >= 0) pyn = __ldcg(w + cv1.y);
      if (qn + nthr < np) cv2 = ldg2i_hint(code + 2 * (qn + nthr), pol_s);
    }
    double2 wv;
    gs_point_seg(cv.x, av.x, px, 0, av.x, wv.x, rcp_tab);
    gs_point_seg(cv.y, av.y, py, 0, av.y, wv.y, rcp_tab);
    double xd = 0.0;
    upd_point<true>(alpha, xd, rv.x, 0.0, av.x, dv.x, wv.x, hz, acc);
    upd_point<true>(alpha, xd, rv.y, 0.0, av.y, dv.y, wv.y, hz, acc);
    st2_hint(r + 2 * q, rv, pol_r);
    cv = cv1;
    cv1 = cv2;
    dv = dvn;
    rv = rvn;
    av = avn;
    px = pxn;
    py = pyn;
  }
  if ((n & 1) && gtid == 0) {
    const int64_t t = n - 1;
    double xd = 0.0, at = 0.0, wq = 0.0;
    const int32_t c = code[t];
    const double pt = c >= 0 ? __ldcg(w + c) : 0.0;
    gs_point_seg(c, __ldcg(w + t), pt, 0, at, wq, rcp_tab);
    upd_point<true>(alpha, xd, r[t], 0.0, at, hz ? invD[t] : 0.0, wq, hz, acc);
  }
  double v[3] = {acc.rr, acc.rz, acc.zap};
  block_sum<3>(v, red);
  const int nb = gridDim.x;
  if (threadIdx.x == 0) {
    partials[0 * kVecMaxBlocks + blockIdx.x] = v[0];
    partials[1 * kVecMaxBlocks + blockIdx.x] = v[1];
    partials[2 * kVecMaxBlocks + blockIdx.x] = v[2];
  }
  if (last_block(&st->ticket[1], nb)) {
    double sres[3];
    reduce_partials<3>(partials, nb, kVecMaxBlocks, sres, red);
    if (threadIdx.x == 0) {
      st->rr = sres[0];
      if (hz) st->rz_new = sres[1];
      st->zap = sres[2];
      st->alpha = alpha;
      st->iter = st->iter + 1;
    }
  }
}

static bool gs_pre_resident(int64_t g) {
  static int per = -1, sms = 0;
  if (per < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cg_update_gs_pre_kernel, kVecThreads,
                                                      0) != cudaSuccess)
      per = 0;
  }
  return (int64_t)per * sms >= g;   // the barrier needs the whole grid resident
}

extern "C" int nk_cg_update_gs_cls_fused(int64_t n) {
  return (knob(NK_KNOB_GS_TAIL) == 2 && (cg_pipe(n) & 3) == 2 && gs_pre_resident(vec_grid(n)))
             ? 1 : 0;
}

extern "C" int nk_cg_update_gs_cls(int64_t n, double* r, double* w, const double* invD,
                                   const int32_t* code, int nclass, const int32_t* sizes,
                                   const int64_t* nsegs, const int32_t* const* members,
                                   nk_cg_state* st, double* partials, nk_stream_t stream) {
  if (n < 0 || !r || !w || !code || !st || !partials) {
    set_error("cg_update_gs_cls: invalid arguments");
    return NK_ERR_INVALID;
  }
  GsTail T{};
  int rc = gs_tail_build(T, nclass, sizes, nsegs, members);
  if (rc != NK_OK) return rc;
  bool fuse = T.n > 0 && knob(NK_KNOB_GS_TAIL) == 2 && aligned16(r, w, invD) &&
              ((uintptr_t)code & 7) == 0 && (cg_pipe(n) & 3) == 2;
  const int64_t g = vec_grid(n);
  if (fuse) fuse = gs_pre_resident(g);
  if (!fuse) {
    if (T.n > 0) {
      rc = nk_gs_op_classes(nclass, sizes, nsegs, members, w, NK_OP_ADD, 1, 0, st, stream);
      if (rc != NK_OK) return rc;
    }
    return nk_cg_update_gs(n, r, w, invD, code, st, partials, stream);
  }
  launch_ex(kPdlVec, cg_update_gs_pre_kernel, dim3((unsigned)g), dim3(kVecThreads), 0, S(stream),
            n, r, w, invD, code, st, partials, T, knob(NK_KNOB_CG_UPDATE), knob(NK_KNOB_L2));
  return check_launch("cg_update_gs_pre");
}

extern "C" int nk_cg_pupdate(int64_t n, const double* r, double* p, const double* invD,
                             const double* z, nk_cg_state* st, double* hist, nk_stream_t stream) {
  if (n < 0 || !r || !p || !st) {
    set_error("cg_pupdate: invalid arguments");
    return NK_ERR_INVALID;
  }
  if (aligned16(r, p, invD, z))
    cg_pupdate_kernel<true><<<(unsigned)vec_grid(n), kVecThreads, 0, S(stream)>>>(n, r, p, invD, z,
                                                                                st, hist);
  else
    cg_pupdate_kernel<false><<<(unsigned)vec_grid(n), kVecThreads, 0, S(stream)>>>(n, r, p, invD,
                                                                                 z, st, hist);
  return check_launch("cg_pupdate");
}

// The vector head of the fused BP5 step (bk5_pcg.cuh, nk_bk5_pcg) as its own
// coalesced pass: at iteration k = st->iter, k > 0: test ||r_k||, x += alpha_{k-1}
// p_{k-1}, p_k = invD r_k + beta_k p_{k-1}; the last block records hist[k] and
// the stop / rz bookkeeping exactly as nk_bk5_pcg's last block does.  Followed
// by nk_bk5 with st (w = mask A p, st->pAp) it replaces nk_bk5_pcg at orders
// where the fused kernel's row-wise prologue is latency-bound (N != 7).
// Batched: gridDim.y components, component c at c * cstride in x / r / p,
// state st + c, history hist + c * hstride (invD shared).
template <bool VEC>
__global__ void __launch_bounds__(kVecThreads)
cg_xpstep_kernel(int64_t n, double* __restrict__ x, const double* __restrict__ r,
                 double* __restrict__ p, const double* __restrict__ invD, nk_cg_state* st,
                 double* __restrict__ hist, int64_t cstride = 0, int64_t hstride = 0) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.y) {
    x += blockIdx.y * cstride;
    r += blockIdx.y * cstride;
    p += blockIdx.y * cstride;
    st += blockIdx.y;
    if (hist) hist += blockIdx.y * hstride;
  }
  if (st->done) return;
  const int it = st->iter;
  const bool conv = it > 0 && st->rr <= st->thresh2;
  const bool stop = it > 0 && (conv || it >= st->max_iter);
  const double alpha_prev = st->alpha;
  const double rz = st->rz;
  const double beta =
      it == 0 ? 0.0 : (st->flexible ? (-alpha_prev * st->zap) / rz : st->rz_new / rz);
  if (it > 0) {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    if (VEC) {
      const int64_t np = n >> 1;
#pragma unroll 2
      for (int64_t q = gtid; q < np; q += nthr) {
        const double2 pv = reinterpret_cast<const double2*>(p)[q];
        double2 xv = reinterpret_cast<const double2*>(x)[q];
        xv.x = fma(alpha_prev, pv.x, xv.x);
        xv.y = fma(alpha_prev, pv.y, xv.y);
        reinterpret_cast<double2*>(x)[q] = xv;
        if (!stop) {
          const double2 rv = __ldg(reinterpret_cast<const double2*>(r) + q);
          const double2 dv = __ldg(reinterpret_cast<const double2*>(invD) + q);
          reinterpret_cast<double2*>(p)[q] =
              make_double2(fma(beta, pv.x, dv.x * rv.x), fma(beta, pv.y, dv.y * rv.y));
        }
      }
      if ((n & 1) && gtid == 0) {
        const int64_t q = n - 1;
        const double pv = p[q];
        x[q] = fma(alpha_prev, pv, x[q]);
        if (!stop) p[q] = fma(beta, pv, invD[q] * r[q]);
      }
    } else {
      for (int64_t q = gtid; q < n; q += nthr) {
        const double pv = p[q];
        x[q] = fma(alpha_prev, pv, x[q]);
        if (!stop) p[q] = fma(beta, pv, invD[q] * r[q]);
      }
    }
  }
  if (last_block(&st->ticket[2], gridDim.x)) {
    if (threadIdx.x == 0) {
      if (it > 0 && hist) hist[it] = sqrt(st->rr);
      if (stop) {
        st->converged = conv ? 1 : 0;
        st->done = 1;
      } else if (it > 0) {
        st->rz = st->rz_new;
      }
    }
  }
}

extern "C" int nk_cg_xpstep_batch(int64_t n, int ncomp, int64_t cstride, double* x,
                                  const double* r, double* p, const double* invD,
                                  nk_cg_state* st, double* hist, int64_t hstride,
                                  nk_stream_t stream) {
  if (n < 0 || ncomp < 1 || ncomp > 65535 || (ncomp > 1 && cstride < n) || !x || !r || !p ||
      !invD || !st) {
    set_error("cg_xpstep: invalid arguments");
    return NK_ERR_INVALID;
  }
  const dim3 g((unsigned)vec_grid(n), (unsigned)ncomp);
  if (aligned16(x, r, p, invD) && (cstride % 2 == 0 || ncomp == 1))
    launch_ex(kPdlVec, cg_xpstep_kernel<true>, g, dim3(kVecThreads), 0, S(stream), n, x, r, p,
              invD, st, hist, cstride, hstride);
  else
    launch_ex(kPdlVec, cg_xpstep_kernel<false>, g, dim3(kVecThreads), 0, S(stream), n, x, r, p,
              invD, st, hist, cstride, hstride);
  return check_launch("cg_xpstep");
}

extern "C" int nk_cg_xpstep(int64_t n, double* x, const double* r, double* p,
                            const double* invD, nk_cg_state* st, double* hist,
                            nk_stream_t stream) {
  return nk_cg_xpstep_batch(n, 1, 0, x, r, p, invD, st, hist, 0, stream);
}

template <bool VEC>
__global__ void __launch_bounds__(kVecThreads)
pointwise_kernel(int64_t n, const double* a, const double* b, double* y, double alpha,
                 const uint8_t* __restrict__ mask) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  if (VEC) {
    const int64_t np = n >> 1;
    for (int64_t q = gtid; q < np; q += nthr) {
      const double2 av = reinterpret_cast<const double2*>(a)[q];
      const double2 bv = reinterpret_cast<const double2*>(b)[q];
      double2 yv = make_double2(alpha * av.x * bv.x, alpha * av.y * bv.y);
      if (mask) {
        const uchar2 mv = reinterpret_cast<const uchar2*>(mask)[q];
        yv.x = mv.x ? yv.x : 0.0;
        yv.y = mv.y ? yv.y : 0.0;
      }
      reinterpret_cast<double2*>(y)[q] = yv;
    }
    if ((n & 1) && gtid == 0) {
      const int64_t q = n - 1;
      y[q] = (mask && !mask[q]) ? 0.0 : alpha * a[q] * b[q];
    }
  } else {
    for (int64_t q = gtid; q < n; q += nthr) y[q] = (mask && !mask[q]) ? 0.0 : alpha * a[q] * b[q];
  }
}

__global__ void cg_gate_kernel(nk_cg_state* inner, const nk_cg_state* outer) {
  if (outer->done) inner->done = 1;
}

extern "C" int nk_cg_gate(nk_cg_state* inner, const nk_cg_state* outer, nk_stream_t stream) {
  if (!inner || !outer) {
    set_error("cg_gate: invalid arguments");
    return NK_ERR_INVALID;
  }
  cg_gate_kernel<<<1, 1, 0, S(stream)>>>(inner, outer);
  return check_launch("cg_gate");
}

extern "C" int nk_pointwise(int64_t n, const double* a, const double* b, double* y,
                            double alpha, const uint8_t* mask, nk_stream_t stream) {
  if (n < 0 || !a || !b || !y) {
    set_error("pointwise: invalid arguments");
    return NK_ERR_INVALID;
  }
  if (n == 0) return NK_OK;
  const unsigned g = (unsigned)vec_grid(n);
  if (aligned16(a, b, y) && ((uintptr_t)mask & 1) == 0)
    pointwise_kernel<true><<<g, kVecThreads, 0, S(stream)>>>(n, a, b, y, alpha, mask);
  else
    pointwise_kernel<false><<<g, kVecThreads, 0, S(stream)>>>(n, a, b, y, alpha, mask);
  return check_launch("pointwise");
}

extern "C" int nk_wdot(int64_t n, const double* a, const double* b, const double* wt,
                       double* out, double* partials, nk_stream_t stream) {
  if (n < 0 || !a || !b || !out || !partials) {
    set_error("wdot: invalid arguments");
    return NK_ERR_INVALID;
  }
  const int64_t g = vec_grid(n);
  cudaStream_t s = S(stream);
  wdot_partial_kernel<<<(unsigned)g, kVecThreads, 0, s>>>(n, a, b, wt, partials);
  int rc = check_launch("wdot_partial");
  if (rc) return rc;
  wdot_final_kernel<<<1, kVecThreads, 0, s>>>(g, partials, out);
  return check_launch("wdot_final");
}
