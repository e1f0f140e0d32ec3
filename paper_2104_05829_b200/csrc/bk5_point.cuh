// BK5 at N = 2 (NQ = 3, 27-point elements): one THREAD PER POINT, 16
// elements per 432-thread CTA, two CTAs per SM, nk_bk5 variant 11.
//
// At N + 1 = 3 a pencil is 3 points: the pencil kernels put 9 threads on an
// element and move its 216-byte u and 1296-byte G through many tiny strided
// accesses (pencil2: 75% of HBM peak).  Here every access of the streamed
// operands is the point's own, so all of them are warp-coalesced: u (one
// double per thread) is staged into shared memory for the three forward
// contractions (9 reads, D-hat from the constant bank), the six G components
// are six coalesced loads per thread, gr / gs / gt go through shared memory
// for the three backward contractions, and w leaves as one coalesced store.
// Same algorithm as the pencil kernels (w = D^T G D u, PAPER.md BK5),
// different summation order (rounding-level differences).
// The fused p.Ap (split BP5 step) reduces one partial per persistent CTA.
#pragma once

namespace nk {

constexpr int kPtEPB = 8;                  // elements per group
constexpr int kPtThreads = kPtEPB * 27;    // 216 threads, four CTAs per SM
constexpr int kPtPerSM = 4;
constexpr int kPtNS = 3;                   // staged groups in flight
constexpr int kPtStage = kPtEPB * 27 * 7;  // doubles per stage: u | G[6]

// Persistent CTAs (two per SM); the group's u and G (24 KB, contiguous for a
// whole-array call) are moved by one thread with cp.async.bulk into a
// three-stage shared ring, so two groups are always in flight while one
// computes.  A partial last group whose u bytes are not a 16-byte multiple
// copies one double less and loads it directly.
template <int NQ_ = 3>   // a template so every translation unit may include it
__global__ void __launch_bounds__(kPtThreads, kPtPerSM)
bk5_point3(int64_t nlist, const __grid_constant__ DParam<3> D, const double* __restrict__ G,
           const double* __restrict__ u, double* __restrict__ w, double lam0,
           const double* __restrict__ B, double lam1, const uint8_t* __restrict__ mask,
           nk_cg_state* st, double* __restrict__ partials, int64_t part_base,
           int64_t reduce_count) {
  constexpr int NQ = 3, NP = 27, T = kPtThreads;
  extern __shared__ __align__(128) double smem[];
  double* sr = smem + kPtNS * kPtStage;
  double* ss = sr + T;
  double* st3 = ss + T;
  double* red = st3 + T;
  double* sD = red + 32;   // D-hat: lanes of a warp index different rows, which
                           // the constant cache would serialize; shared memory
                           // serves the distinct words in one wavefront
  uint64_t* bar = reinterpret_cast<uint64_t*>(sD + 10);   // [kPtNS]
  if (st != nullptr && st->done) return;
  const int t = threadIdx.x;
  if (t < 9) sD[t] = D.d[t];
  __syncthreads();
  // this point's D-hat rows (forward) and columns (backward) in registers:
  // 18 shared reads per point and group otherwise (MIO-throttle bound)
  double di[NQ], dj[NQ], dk[NQ], ti[NQ], tj[NQ], tk[NQ];
  const int le = t / NP, p = t - le * NP;
  const int i = p % NQ, j = (p / NQ) % NQ, k = p / (NQ * NQ);
  const int base = le * NP;
#pragma unroll
  for (int m = 0; m < NQ; ++m) {
    di[m] = sD[i * NQ + m];
    dj[m] = sD[j * NQ + m];
    dk[m] = sD[k * NQ + m];
    ti[m] = sD[m * NQ + i];
    tj[m] = sD[m * NQ + j];
    tk[m] = sD[m * NQ + k];
  }
  const int64_t ngroups = (nlist + kPtEPB - 1) / kPtEPB;
  auto issue = [&](int64_t grp, int s) {
    const int64_t e0 = grp * kPtEPB;
    const int64_t cnt = nlist - e0 < kPtEPB ? nlist - e0 : kPtEPB;
    double* dst = smem + s * kPtStage;
    const uint32_t ub = (uint32_t)(cnt * NP * sizeof(double)) & ~15u;
    const uint32_t gb = (uint32_t)(cnt * 6 * NP * sizeof(double));
    mbar_expect_tx(&bar[s], ub + gb);
    tma_load_1d(dst, u + e0 * NP, ub, &bar[s]);
    tma_load_1d(dst + T, G + e0 * 6 * NP, gb, &bar[s]);
  };
  if (t == 0) {
    for (int q = 0; q < kPtNS; ++q) mbar_init(&bar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < kPtNS; ++q)
      if ((int64_t)blockIdx.x + q * gridDim.x < ngroups) issue(blockIdx.x + q * gridDim.x, q);
  }
  __syncthreads();
  double dot = 0.0;
  int it = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int s = it % kPtNS;
    const double* su = smem + s * kPtStage;
    const double* sg = su + T;
    const int64_t e0 = grp * kPtEPB;
    const int cnt = (int)(nlist - e0 < kPtEPB ? nlist - e0 : kPtEPB);
    const bool act = le < cnt;
    const int64_t q = (e0 + le) * NP + p;
    mbar_wait(&bar[s], (it / kPtNS) & 1);
    // the double a 16-byte-rounded u copy left out (odd cnt): read directly
    const bool odd_tail = (cnt & 1) && t == cnt * NP - 1;
    const double uv = act ? (odd_tail ? u[q] : su[t]) : 0.0;
    double ur = 0.0, us = 0.0, ut = 0.0;
    if (act) {
#pragma unroll
      for (int m = 0; m < NQ; ++m) {
        const int qi = base + k * 9 + j * 3 + m, qj = base + k * 9 + m * 3 + i,
                  qk = base + m * 9 + j * 3 + i;
        const int tail = cnt * NP - 1;
        ur = fma(di[m], (cnt & 1) && qi == tail ? u[e0 * NP + qi] : su[qi], ur);
        us = fma(dj[m], (cnt & 1) && qj == tail ? u[e0 * NP + qj] : su[qj], us);
        ut = fma(dk[m], (cnt & 1) && qk == tail ? u[e0 * NP + qk] : su[qk], ut);
      }
      const double* gp = sg + le * 6 * NP + p;
      const double g0 = gp[0], g1 = gp[NP], g2 = gp[2 * NP], g3 = gp[3 * NP], g4 = gp[4 * NP],
                   g5 = gp[5 * NP];
      sr[t] = g0 * ur + g1 * us + g2 * ut;
      ss[t] = g1 * ur + g3 * us + g4 * ut;
      st3[t] = g2 * ur + g4 * us + g5 * ut;
    }
    __syncthreads();   // (A) stage s read for the last time; gr / gs / gt complete
    if (t == 0 && grp + kPtNS * (int64_t)gridDim.x < ngroups)
      issue(grp + kPtNS * (int64_t)gridDim.x, s);
    if (act) {
      double wv = 0.0;
#pragma unroll
      for (int m = 0; m < NQ; ++m) {
        wv = fma(ti[m], sr[base + k * 9 + j * 3 + m], wv);
        wv = fma(tj[m], ss[base + k * 9 + m * 3 + i], wv);
        wv = fma(tk[m], st3[base + m * 9 + j * 3 + i], wv);
      }
      double res = lam0 * wv;
      if (B != nullptr) res = fma(lam1 * __ldg(B + q), uv, res);
      if (mask != nullptr) res = mask[q] ? res : 0.0;
      if (st != nullptr) dot = fma(uv, res, dot);
      w[q] = res;
    }
    __syncthreads();   // (B) gr / gs / gt free for the next group
  }
  if (st != nullptr) {
    double vv[1] = {dot};
    block_sum<1>(vv, red);
    if (t == 0) partials[part_base + blockIdx.x] = vv[0];
    if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) {
      double sres[1];
      reduce_partials<1>(partials, reduce_count, 0, sres, red);
      if (t == 0) st->pAp = sres[0];
    }
  }
}

inline size_t point3_smem() {
  return sizeof(double) * ((size_t)kPtNS * kPtStage + 3 * kPtThreads + 32 + 10) +
         kPtNS * sizeof(uint64_t);
}

inline int64_t point3_blocks(int64_t nlist) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(bk5_point3<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)point3_smem());
  }
  const int64_t ng = (nlist + kPtEPB - 1) / kPtEPB;
  return ng < kPtPerSM * sms ? ng : kPtPerSM * sms;
}

// whole-array calls only (contiguous element groups): u and G 16-byte aligned
inline int launch_point3(int64_t nlist, const double* Dhost, const double* G, const double* u,
                         double* w, double lam0, const double* B, double lam1,
                         const uint8_t* mask, nk_cg_state* st, double* partials,
                         int64_t part_base, int64_t reduce_count, cudaStream_t s) {
  const int64_t nb = point3_blocks(nlist);
  if (nb == 0) return NK_OK;
  DParam<3> D;
  D.set(Dhost);
  bk5_point3<3><<<(unsigned)nb, kPtThreads, point3_smem(), s>>>(nlist, D, G, u, w, lam0, B, lam1,
                                                              mask, st, partials, part_base,
                                                              reduce_count);
  return check_launch("bk5_point3");
}

}  // namespace nk
