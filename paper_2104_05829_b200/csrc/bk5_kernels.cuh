// BK5: element-local spectral-element stiffness (+ mass) apply on sm_100a.
//
//   w_e = lam0 * [D1;D2;D3]^T G_e [D1;D2;D3] u_e + lam1 * B_e u_e
//
// SPEC.md:370-378 (apply_stiffness_local), PAPER.md:1150-1162 (contractions
// u_r[k,j,i] = sum_m D[i,m] u[k,j,m], u_s along j, u_t along k) and
// PAPER.md:1240-1266 (six symmetric factors, 12(N+1)^4 + 15(N+1)^3 flops).
//
// Variant 1, "k-slab": one (N+1)x(N+1) thread plane per element (the paper's
// 2D thread structure).  Thread (i,j) keeps its k-column of
// u and of G_t u in registers, so the t-direction contractions never touch
// shared memory; the r/s contractions read a padded shared copy of the
// element (conflict-free row stride NQ|1).  Several elements per CTA so the
// CTA has ~256 threads.  Every global access is a coalesced plane of the
// element (consecutive threads -> consecutive points).  HBM traffic per
// point: u 8 B + G 48 B + w 8 B (+ B 8 B, + mask 1 B).
//
#pragma once
#include "common.cuh"

namespace nk {

// D-hat as a kernel parameter (constant bank), plus its even-odd split.
// D-hat is centro-antisymmetric (D[N-q][N-m] = -D[q][m]: GLL nodes are
// symmetric), and so is its transpose; with s_m = v_m + v_{N-m},
// d_m = v_m - v_{N-m} (m < H = NQ/2) a 1-D derivative is
//   out_q = O_q + E_q,  out_{N-q} = O_q - E_q  (q < H),  out_mid = M . d  (NQ odd)
//   E_q = sum_m Ev[q][m] s_m (+ Ev[q][H] v_mid),  O_q = sum_m Od[q][m] d_m
// with Ev = (D[q][m] + D[q][N-m]) / 2 (Ev[q][H] = D[q][mid]), Od = (D[q][m] -
// D[q][N-m]) / 2, M[m] = D[mid][m]: about half the multiply-adds and half the
// D-hat operand fetches of the direct product (the rounding differs from it
// at the 1e-16 level).  eo holds the forward tables, then the transposed ones.
// Every table row starts on an even index and the struct is 16-byte aligned
// with eo first, so consecutive coefficient pairs (m, m+1), m even, sit in one
// 16-byte constant-bank chunk: one LDCU.128 feeds two DFMAs without uniform-
// register shuffles (rows of odd length H + ODD or H used to straddle chunks).
template <int NQ>
struct alignas(16) DParam {
  static constexpr int H = NQ / 2, ODD = NQ & 1, HE = H + ODD;
  static constexpr int SE = (HE + 1) & ~1, SO = (H + 1) & ~1;   // even row strides
  static constexpr int OO = H * SE, OM = OO + H * SO;           // O rows, middle row
  static constexpr int EOF_ = (OM + ODD * H + 1) & ~1;          // one direction (even)
  __host__ __device__ static constexpr int ei(int q, int m) { return q * SE + m; }
  __host__ __device__ static constexpr int oi(int q, int m) { return OO + q * SO + m; }
  __host__ __device__ static constexpr int mi(int m) { return OM + m; }
  double eo[2 * EOF_ > 0 ? 2 * EOF_ : 2];
  double d[NQ * NQ];   // row-major D[a][m] = h_m'(xi_a)
  void set(const double* Dh) {   // host
    for (int q = 0; q < NQ * NQ; ++q) d[q] = Dh[q];
    for (int q = 0; q < (2 * EOF_ > 0 ? 2 * EOF_ : 2); ++q) eo[q] = 0.0;
    for (int tr = 0; tr < 2; ++tr) {
      double* T = eo + tr * EOF_;
      auto A = [&](int q, int m) { return tr ? Dh[m * NQ + q] : Dh[q * NQ + m]; };
      for (int q = 0; q < H; ++q) {
        for (int m = 0; m < H; ++m) {
          T[ei(q, m)] = 0.5 * (A(q, m) + A(q, NQ - 1 - m));
          T[oi(q, m)] = 0.5 * (A(q, m) - A(q, NQ - 1 - m));
        }
        if (ODD) T[ei(q, H)] = A(q, H);
      }
      if (ODD)
        for (int m = 0; m < H; ++m) T[mi(m)] = A(H, m);
    }
  }
};

// Tunable shape: EPB elements per CTA (EPB*NQ^2 threads), MINB CTAs per SM
// requested from ptxas (register cap 65536 / (MINB * threads)).
template <int NQ, int EPB_ = ((256 / (NQ * NQ)) > 0 ? (256 / (NQ * NQ)) : 1),
          int MINB_ = (NQ <= 8 ? 2 : 1)>
struct Bk5Cfg {
  static constexpr int NQ2 = NQ * NQ;
  static constexpr int NQ3 = NQ * NQ * NQ;
  static constexpr int EPB = EPB_;
  static constexpr int THREADS = EPB * NQ2;
  static constexpr int MINB = MINB_;
  static constexpr int NQP = (NQ % 2 == 0) ? NQ + 1 : NQ;  // padded row stride
  static constexpr int PLANE = NQ * NQP;
  static constexpr int VOL = NQ * PLANE;
  static size_t smem_bytes(int nc) {
    return sizeof(double) * (size_t)(2 * NQ * NQP + (size_t)EPB * 3 * nc * VOL + 32);
  }
};

template <int NQ, int NC, int EPB, int MINB>
__global__ void __launch_bounds__(EPB * NQ * NQ, MINB)
bk5_kslab(int64_t nlist, const int32_t* __restrict__ elist, const __grid_constant__ DParam<NQ> Dg,
          const double* __restrict__ G, const double* __restrict__ u, double* __restrict__ w,
          double lam0, const double* __restrict__ B, double lam1, int64_t cstride,
          const uint8_t* __restrict__ mask, nk_cg_state* st, double* __restrict__ partials,
          int64_t part_base, int64_t reduce_count, int pf_dist) {
  using C = Bk5Cfg<NQ, EPB, MINB>;
  constexpr int NQ2 = C::NQ2, NQ3 = C::NQ3, NQP = C::NQP, PLANE = C::PLANE, VOL = C::VOL;
  extern __shared__ double smem[];
  if (st != nullptr && st->done) return;

  const int t = threadIdx.x;
  // L2 prefetch for the block that will run ~pf_dist blocks later (about one
  // wave ahead): DRAM streaming no longer waits on this block's load latency.
  if (pf_dist > 0 && t == 0) {
    const int64_t nb = (int64_t)blockIdx.x + pf_dist;
    const int64_t s0 = nb * EPB;
    if (s0 < nlist) {
      const int64_t s1 = s0 + EPB < nlist ? s0 + EPB : nlist;
      if (elist == nullptr) {
        prefetch_l2(G + s0 * 6 * NQ3, (s1 - s0) * 6 * NQ3 * (int64_t)sizeof(double));
        for (int c = 0; c < NC; ++c)
          prefetch_l2(u + c * cstride + s0 * NQ3, (s1 - s0) * NQ3 * (int64_t)sizeof(double));
      } else {
        for (int64_t q = s0; q < s1; ++q) {
          const int64_t e = elist[q];
          prefetch_l2(G + e * 6 * NQ3, 6 * NQ3 * (int64_t)sizeof(double));
          for (int c = 0; c < NC; ++c)
            prefetch_l2(u + c * cstride + e * NQ3, NQ3 * (int64_t)sizeof(double));
        }
      }
    }
  }

  double* sD = smem;              // sD[a*NQP+m]  = D[a][m]
  double* sDt = sD + NQ * NQP;    // sDt[a*NQP+m] = D[m][a]
  double* red = sDt + NQ * NQP;   // 32 doubles for the fused dot
  double* sel = red + 32;

  const int le = t / NQ2;
  const int ij = t - le * NQ2;
  const int i = ij % NQ, j = ij / NQ;
  for (int q = t; q < NQ * NQ; q += blockDim.x) {
    const int a = q / NQ, m = q - (q / NQ) * NQ;
    const double d = Dg.d[q];
    sD[a * NQP + m] = d;
    sDt[m * NQP + a] = d;
  }

  const int64_t slot = (int64_t)blockIdx.x * C::EPB + le;
  const bool active = slot < nlist;
  const int64_t e = active ? (elist ? (int64_t)elist[slot] : slot) : 0;
  double* su = sel + (size_t)le * 3 * NC * VOL;  // [NC][VOL]
  double* sgr = su + NC * VOL;                    // [NC][VOL]
  double* sgs = sgr + NC * VOL;                   // [NC][VOL]

  const int64_t ebase = e * NQ3 + ij;
  double ru[NC][NQ];
  if (active) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        ru[c][k] = __ldg(u + c * cstride + ebase + k * NQ2);
        su[c * VOL + k * PLANE + j * NQP + i] = ru[c][k];
      }
  }
  __syncthreads();

  double rgt[NC][NQ];
  if (active) {
    const double* gp = G + e * 6 * NQ3 + ij;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const double g0 = __ldg(gp + 0 * NQ3 + k * NQ2);
      const double g1 = __ldg(gp + 1 * NQ3 + k * NQ2);
      const double g2 = __ldg(gp + 2 * NQ3 + k * NQ2);
      const double g3 = __ldg(gp + 3 * NQ3 + k * NQ2);
      const double g4 = __ldg(gp + 4 * NQ3 + k * NQ2);
      const double g5 = __ldg(gp + 5 * NQ3 + k * NQ2);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double* uk = su + c * VOL + k * PLANE;
        double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
          ur = fma(sD[i * NQP + m], uk[j * NQP + m], ur);
          us = fma(sD[j * NQP + m], uk[m * NQP + i], us);
          ut = fma(sD[k * NQP + m], ru[c][m], ut);
        }
        sgr[c * VOL + k * PLANE + j * NQP + i] = g0 * ur + g1 * us + g2 * ut;
        sgs[c * VOL + k * PLANE + j * NQP + i] = g1 * ur + g3 * us + g4 * ut;
        rgt[c][k] = g2 * ur + g4 * us + g5 * ut;
      }
    }
  }
  __syncthreads();

  double dot = 0.0;
  if (active) {
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int64_t gi = ebase + k * NQ2;
      const bool keep = mask ? (mask[gi] != 0) : true;
      const double bm = B ? lam1 * __ldg(B + gi) : 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double* grk = sgr + c * VOL + k * PLANE;
        const double* gsk = sgs + c * VOL + k * PLANE;
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < NQ; ++m) {
          acc = fma(sDt[i * NQP + m], grk[j * NQP + m], acc);
          acc = fma(sDt[j * NQP + m], gsk[m * NQP + i], acc);
          acc = fma(sDt[k * NQP + m], rgt[c][m], acc);
        }
        const double uv = su[c * VOL + k * PLANE + j * NQP + i];
        acc = lam0 * acc + bm * uv;
        acc = keep ? acc : 0.0;
        w[c * cstride + gi] = acc;
        dot = fma(uv, acc, dot);
      }
    }
  }

  if (st != nullptr) {
    double v[1] = {dot};
    block_sum<1>(v, red);
    if (t == 0) partials[part_base + blockIdx.x] = v[0];
    if (reduce_count > 0 && last_block(&st->ticket[0], gridDim.x)) {
      double s[1];
      reduce_partials<1>(partials, reduce_count, 0, s, red);
      if (t == 0) st->pAp = s[0];
    }
  }
}

template <int NQ, int NC, int EPB = Bk5Cfg<NQ>::EPB, int MINB = Bk5Cfg<NQ>::MINB>
static int launch_kslab(int64_t nlist, const int32_t* elist, const double* Dhost, const double* G,
                        const double* u, double* w, double lam0, const double* B, double lam1,
                        int64_t cstride, const uint8_t* mask, nk_cg_state* st, double* partials,
                        int64_t part_base, int64_t reduce_count, cudaStream_t s, int pf_dist) {
  using C = Bk5Cfg<NQ, EPB, MINB>;
  const size_t smem = C::smem_bytes(NC);
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(bk5_kslab<NQ, NC, EPB, MINB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) {
      set_error("bk5: smem attribute (%zu B): %s", smem, cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  const int64_t nblk = (nlist + C::EPB - 1) / C::EPB;
  if (nblk == 0) return NK_OK;
  DParam<NQ> D;
  D.set(Dhost);
  bk5_kslab<NQ, NC, EPB, MINB><<<(unsigned)nblk, C::THREADS, smem, s>>>(
      nlist, elist, D, G, u, w, lam0, B, lam1, cstride, mask, st, partials, part_base,
      reduce_count, pf_dist);
  return check_launch("bk5_kslab");
}

template <int NQ, int EPB = Bk5Cfg<NQ>::EPB>
static int64_t kslab_blocks(int64_t nlist) {
  return (nlist + EPB - 1) / EPB;
}

// ---------------------------------------------------------------- local diag
// diag[k,j,i] = sum_m D[m,i]^2 G11[k,j,m] + sum_m D[m,j]^2 G22[k,m,i]
//             + sum_m D[m,k]^2 G33[m,j,i] + 2 D[i,i]D[j,j] G12 + 2 D[i,i]D[k,k] G13
//             + 2 D[j,j]D[k,k] G23      (then * lam0 + lam1 B)
template <int NQ>
__global__ void local_diag_kernel(int64_t nelem, const double* __restrict__ D,
                                  const double* __restrict__ G, double lam0,
                                  const double* __restrict__ B, double lam1,
                                  double* __restrict__ diag) {
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nelem * NQ3) return;
  const int64_t e = p / NQ3;
  const int r = (int)(p - e * NQ3);
  const int i = r % NQ, j = (r / NQ) % NQ, k = r / NQ2;
  const double* g = G + e * 6 * NQ3;
  double s = 0.0;
  for (int m = 0; m < NQ; ++m) {
    const double a = D[m * NQ + i], b = D[m * NQ + j], c = D[m * NQ + k];
    s += a * a * g[0 * NQ3 + k * NQ2 + j * NQ + m];
    s += b * b * g[3 * NQ3 + k * NQ2 + m * NQ + i];
    s += c * c * g[5 * NQ3 + m * NQ2 + j * NQ + i];
  }
  const double di = D[i * NQ + i], dj = D[j * NQ + j], dk = D[k * NQ + k];
  s += 2.0 * di * dj * g[1 * NQ3 + r] + 2.0 * di * dk * g[2 * NQ3 + r] +
       2.0 * dj * dk * g[4 * NQ3 + r];
  s *= lam0;
  if (B) s += lam1 * B[p];
  diag[p] = s;
}

}  // namespace nk
