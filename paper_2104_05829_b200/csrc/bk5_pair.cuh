// BK5 at N = 15 (NQ = 16) on a CTA PAIR (thread-block cluster of two SMs,
// nk_bk5 variant 10).  Paper: the local stiffness apply w = D^T G D u
// (PAPER.md BK5; SPEC.md apply_stiffness_local); same arithmetic as
// bk5_stage16, different partition.
//
// Why: at N + 1 = 16 one element's operands are u 32 KB + G 192 KB, so a
// single CTA cannot stage all six G components next to its work buffers
// (bk5_stage16 stages four and reads two from L2, which hold 37% of its
// stalls).  Two CTAs of a cluster share ONE element instead, split by
// k-planes: rank c owns the even-odd plane pairs q in [4c, 4c + 4), i.e.
// global planes {q, 15 - q} (rank 0: 0..3, 12..15; rank 1: 4..11), so each
// rank's k-contractions are complete even-odd half matvecs (matvec_half).
//   * u: each rank bulk-loads the two 4-plane chunks it owns with a 2-D
//     tensor copy MULTICAST to both CTAs (.multicast::cluster), so both hold
//     the whole swizzled u (F3 needs full k-columns) while HBM / L2 deliver
//     it once;
//   * G: each rank stages its own 8 planes of all six components (96 KB);
//   * F1 (i-pencils) and F2 (j-pencils) of the rank's 8 planes run on
//     different warps at the same time (128 pencils each); F3 / the G phase /
//     B3 on 256 (j, i) columns, 8 planes each;
//   * B3 needs the whole k-column of gt: the G phase pushes each thread's 8
//     values into the PEER's receive buffer with st.async (asynchronous
//     remote stores that complete on the peer's mbarrier as transaction
//     bytes: no release fence, and the transfer overlaps the G phase);
//   * w is assembled in the rank's own rows of the spent u buffer and leaves
//     by two swizzled tensor stores;
//   * one relaxed cluster barrier per element (after the w stores have read
//     shared memory) orders the buffer reuse across the pair: the peer's
//     multicast of u(next + 1) into this rank's spent u buffer and its next
//     gt pushes into the receive buffer.
// R (the i-derivative, rows swizzled like u) and S (the j-derivative) hold
// the rank's 8 planes.  Shared memory per CTA: 2 x 32 KB u + 96 KB G +
// 16 KB S + 16 KB R + 16 KB receive = 208 KB (one CTA per SM; 74 clusters
// cover the 148 SMs).
#pragma once

namespace nk {

#if defined(NK_BK5_NQ) && NK_BK5_NQ == 16

struct Pair16 {
  static constexpr int NQ = 16, NQ2 = 256, NQ3 = 4096, HP = 8 * NQ2;   // HP: 8 planes
  static constexpr int THREADS = NQ2;
  // (bytes) align slack | U0 | U1 | G[6] (8 planes) | S | R (8 planes) | Xr | red[32] | 4 mbarriers
  static size_t smem_bytes() {
    return 1024 + sizeof(double) * ((size_t)2 * NQ3 + 6 * HP + 3 * HP + 32) +
           4 * sizeof(uint64_t);
  }
  // local plane p (0..7) of rank c -> global k-plane
  __host__ __device__ static constexpr int kglob(int c, int p) {
    return p < 4 ? (c ? 4 : 0) + p : (c ? 8 : 12) + (p - 4);
  }
  // matvec_half output slot j -> local plane (the same for both ranks)
  __host__ __device__ static constexpr int pslot(int j) { return (j & 1) ? 7 - j / 2 : j / 2; }
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
// 16-byte asynchronous store into the peer's shared memory, completing on
// the peer's mbarrier as transaction bytes (dst, bar: shared::cluster
// addresses from mapa)
__device__ __forceinline__ void st_async2(uint32_t dst, double x, double y, uint32_t bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst),
      "d"(x), "d"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int x, int y,
                                               uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// B3 of rank CR: the whole k-column of gt (own slots in registers, the
// peer's from the exchange buffer) -> D^T restricted to this rank's planes
template <int CR>
__device__ __forceinline__ void pair_b3(const DParam<16>& D, const double (&gt)[8],
                                        const double* Xc, int t, double (&o)[8]) {
  double v[16];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[Pair16::kglob(CR, Pair16::pslot(j))] = gt[j];
    v[Pair16::kglob(1 - CR, Pair16::pslot(j))] = Xc[((j >> 1) * 256 + t) * 2 + (j & 1)];
  }
  matvec_half<16, true, CR>(D, v, o);
}

template <bool TRANS>
__device__ __forceinline__ void pair_half(int c, const DParam<16>& D, const double (&v)[16],
                                          double (&o)[8]) {
  if (c == 0)
    matvec_half<16, TRANS, 0>(D, v, o);
  else
    matvec_half<16, TRANS, 1>(D, v, o);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
bk5_pair16(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<16> D,
           const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmw,
           const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ w,
           double lam0, const double* __restrict__ B, double lam1,
           const uint8_t* __restrict__ mask, nk_cg_state* st, double* __restrict__ partials,
           int64_t part_base, int64_t reduce_count) {
  using C = Pair16;
  static_assert(HalfSet<16, 0>::CNT == 8 && HalfSet<16, 1>::CNT == 8, "four pairs per rank");
  constexpr int NQ2 = C::NQ2, NQ3 = C::NQ3, HP = C::HP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (st != nullptr && st->done) return;   // both ranks read the same flag
  // 1024-B aligned (128-byte swizzle atoms), as an offset from smem_raw so
  // that the compiler keeps the shared address space (LDS / STS, not generic
  // LD / ST through the long scoreboard)
  double* Ub0 = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  double* Gb = Ub0 + 2 * NQ3;   // [comp][p][j][i]
  double* Ss = Gb + 6 * HP;     // [p][j][i]
  double* Rr = Ss + HP;         // [p * 16 + j] rows, 16-byte chunks swizzled as u's
  double* Xr = Rr + HP;         // [slot / 2][t][2]: the peer's gt
  double* red = Xr + HP;
  uint64_t* ubar = reinterpret_cast<uint64_t*>(red + 32);   // [2]
  uint64_t* gbar = ubar + 2;
  uint64_t* xbar = ubar + 3;

  const int c = (int)cluster_rank();
  const int peer = c ^ 1;
  const int t = threadIdx.x;
  const int a = t & 15, b = t >> 4;
  // F1 / B1 (warps 0-3: i-pencil of own plane fp, row j = fq) and F2 / B2
  // (warps 4-7: j-pencil of own plane fp, column i = fq)
  const bool row_role = t < 128;
  const int fp = (t & 127) >> 4, fq = t & 15, fk = C::kglob(c, fp);
  const int k0 = c ? 4 : 0, k1 = c ? 8 : 12;   // the two 4-plane chunks
  const int64_t ncl = gridDim.x >> 1;
  const int64_t cid = blockIdx.x >> 1;
  auto elem_of = [&](int64_t slot) -> int64_t { return elist ? (int64_t)elist[slot] : slot; };
  auto issue_u = [&](int64_t slot, int bi) {   // own chunks, multicast to both ranks
    const int row = (int)(elem_of(slot) * NQ2);
    mbar_expect_tx(&ubar[bi], NQ3 * sizeof(double));   // both ranks' halves
    tma_load_2d_mc(Ub0 + bi * NQ3 + k0 * NQ2, &tmu, 0, row + k0 * 16, &ubar[bi], 3);
    tma_load_2d_mc(Ub0 + bi * NQ3 + k1 * NQ2, &tmu, 0, row + k1 * 16, &ubar[bi], 3);
  };
  auto issue_g = [&](int64_t slot) {
    const double* src = G + elem_of(slot) * 6 * NQ3;
    mbar_expect_tx(gbar, 6 * HP * sizeof(double));
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      tma_load_1d(Gb + q * HP, src + q * NQ3 + k0 * NQ2, 4 * NQ2 * sizeof(double), gbar);
      tma_load_1d(Gb + q * HP + 4 * NQ2, src + q * NQ3 + k1 * NQ2, 4 * NQ2 * sizeof(double),
                  gbar);
    }
  };
  if (t == 0) {
    mbar_init(&ubar[0], 1);
    mbar_init(&ubar[1], 1);
    mbar_init(gbar, 1);
    mbar_init(xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();   // both ranks' barriers exist before any multicast lands
  if (t == 0 && cid < nlist) {
    issue_u(cid, 0);
    issue_g(cid);
    if (cid + ncl < nlist) issue_u(cid + ncl, 1);
  }
  const uint32_t xr_peer = peer_addr(Xr, (uint32_t)peer);
  const uint32_t xbar_peer = peer_addr(xbar, (uint32_t)peer);

  double dot = 0.0;
  int it = 0;
  for (int64_t slot = cid; slot < nlist; slot += ncl, ++it) {
    const int64_t e = elem_of(slot);
    const int bi = it & 1;
    double* Uc = Ub0 + bi * NQ3;
    if (t == 0) mbar_expect_tx(xbar, HP * sizeof(double));   // the peer's gt of this element
    mbar_wait(&ubar[bi], (it >> 1) & 1);
    double ut[8];
    {
      double v[16];
      // ---- F3: k-column (j = b, i = a), this rank's 8 output planes
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = Uc[Stage16::sw(m * 16 + b, a)];
      pair_half<false>(c, D, v, ut);
      if (row_role) {   // ---- F1: i-row (k = fk, j = fq) -> R
        const int r = fk * 16 + fq, rr = fp * 16 + fq;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double2 p = *reinterpret_cast<const double2*>(Uc + r * 16 + ((q ^ (r & 7)) << 1));
          v[2 * q] = p.x;
          v[2 * q + 1] = p.y;
        }
        double o[16];
        matvec<16, false>(D, v, o);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<double2*>(Rr + rr * 16 + ((q ^ (rr & 7)) << 1)) =
              make_double2(o[2 * q], o[2 * q + 1]);
      } else {          // ---- F2: j-column (k = fk, i = fq) -> S
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = Uc[Stage16::sw(fk * 16 + m, fq)];
        double o[16];
        matvec<16, false>(D, v, o);
#pragma unroll
        for (int j = 0; j < 16; ++j) Ss[fp * NQ2 + j * 16 + fq] = o[j];
      }
    }
    __syncthreads();   // (A) R, S complete (u is dead from here on)
    mbar_wait(gbar, it & 1);
    double gt[8];
    {  // ---- G: column (b, a) over the 8 own planes (slot order)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int p = C::pslot(j);
        const int k = C::kglob(c, p);
        const int pg = p * NQ2 + b * 16 + a;
        double g[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) g[q] = Gb[q * HP + pg];
        const int qr = Stage16::sw(p * 16 + b, a);
        const double ur = Rr[qr], us = Ss[pg];
        Rr[qr] = g[0] * ur + g[1] * us + g[2] * ut[j];
        Ss[pg] = g[1] * ur + g[3] * us + g[4] * ut[j];
        gt[j] = g[2] * ur + g[4] * us + g[5] * ut[j];
        if (j & 1)
          st_async2(xr_peer + (uint32_t)(((j >> 1) * NQ2 + t) * 2 * sizeof(double)), gt[j - 1],
                    gt[j], xbar_peer);
      }
    }
    __syncthreads();   // (B) G buffer read for the last time
    if (t == 0 && slot + ncl < nlist) issue_g(slot + ncl);
    mbar_wait(xbar, it & 1);   // the peer's gt is in Xr
    double o3[8];
    // ---- B3: column (b, a), D^T over the whole k-column of gt
    if (c == 0)
      pair_b3<0>(D, gt, Xr, t, o3);
    else
      pair_b3<1>(D, gt, Xr, t, o3);
    if (row_role) {   // ---- B1: R row in place
      const int r = fp * 16 + fq;
      double v[16], o[16];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double2 p = *reinterpret_cast<const double2*>(Rr + r * 16 + ((q ^ (r & 7)) << 1));
        v[2 * q] = p.x;
        v[2 * q + 1] = p.y;
      }
      matvec<16, true>(D, v, o);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<double2*>(Rr + r * 16 + ((q ^ (r & 7)) << 1)) =
            make_double2(o[2 * q], o[2 * q + 1]);
    } else {          // ---- B2: S column in place
      double v[16], o[16];
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = Ss[fp * NQ2 + m * 16 + fq];
      matvec<16, true>(D, v, o);
#pragma unroll
      for (int j = 0; j < 16; ++j) Ss[fp * NQ2 + j * 16 + fq] = o[j];
    }
    __syncthreads();   // (C1)
    {  // ---- epilogue: column (b, a), w into the rank's rows of the spent u buffer
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int p = C::pslot(j);
        const int k = C::kglob(c, p);
        const int qr = Stage16::sw(k * 16 + b, a);
        const int64_t off = e * NQ3 + k * NQ2 + b * 16 + a;
        double res = lam0 * (Rr[Stage16::sw(p * 16 + b, a)] + Ss[p * NQ2 + b * 16 + a] + o3[j]);
        if (B != nullptr || st != nullptr) {
          const double uv = __ldg(u + off);
          if (B != nullptr) res = fma(lam1 * __ldg(B + off), uv, res);
          if (mask != nullptr) res = mask[off] ? res : 0.0;
          dot = fma(uv, res, dot);
        } else if (mask != nullptr) {
          res = mask[off] ? res : 0.0;
        }
        Uc[qr] = res;
      }
      fence_proxy_async();
    }
    __syncthreads();   // (C) S free for the next element; w rows in shared
    if (t == 0) {
      tma_store_2d(&tmw, 0, (int)(e * NQ2 + k0 * 16), Uc + k0 * NQ2);
      tma_store_2d(&tmw, 0, (int)(e * NQ2 + k1 * 16), Uc + k1 * NQ2);
      bulk_commit();
      bulk_wait_read0();   // w has left this u buffer
    }
    // (H) both ranks: u buffer bi free (w read out), Xr consumed -- the pair
    // may refill them
    cluster_sync_relaxed();
    if (t == 0 && slot + 2 * ncl < nlist) issue_u(slot + 2 * ncl, bi);
  }
  if (t == 0) bulk_wait0();
  cluster_sync_all();   // no rank leaves while the peer may still address it

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

inline int64_t pair16_grid(int64_t nlist) {
  static int64_t clusters = -1;
  if (clusters < 0) {
    cudaFuncSetAttribute(bk5_pair16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Pair16::smem_bytes());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 148);
    cfg.blockDim = dim3(Pair16::THREADS);
    cfg.dynamicSmemBytes = Pair16::smem_bytes();
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, bk5_pair16, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 74;
    }
    clusters = n;
  }
  return 2 * (nlist < clusters ? nlist : clusters);
}

// u and w must be 16-byte aligned (tensor maps); u_len doubles in u and w.
inline int launch_pair16(int64_t nlist, const int32_t* elist, const double* Dhost,
                         const double* G, const double* u, double* w, double lam0,
                         const double* B, double lam1, const uint8_t* mask, nk_cg_state* st,
                         double* partials, int64_t part_base, int64_t reduce_count,
                         int64_t u_len, cudaStream_t s) {
  const int64_t grid = pair16_grid(nlist);
  if (grid == 0) return NK_OK;
  if (((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(w) |
        reinterpret_cast<uintptr_t>(G)) & 15) || (u_len % 16) != 0) {
    set_error("bk5_pair (N = 15): u, w and G must be 16-byte aligned");
    return NK_ERR_INVALID;
  }
  CUtensorMap tmu, tmw;
  int rc = encode_rows16(&tmu, u, u_len, 64);
  if (rc == NK_OK) rc = encode_rows16(&tmw, w, u_len, 64);
  if (rc != NK_OK) return rc;
  DParam<16> D;
  D.set(Dhost);
  bk5_pair16<<<(unsigned)grid, Pair16::THREADS, Pair16::smem_bytes(), s>>>(
      nlist, elist, D, tmu, tmw, G, u, w, lam0, B, lam1, mask, st, partials, part_base,
      reduce_count);
  return check_launch("bk5_pair16");
}

#endif  // NK_BK5_NQ == 16

}  // namespace nk
