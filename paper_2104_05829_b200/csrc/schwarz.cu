// Overlapping Schwarz smoothing with fast-diagonalisation local solves
// (SPEC.md:410-418 fdm_local_solve, 499-507
// schwarz_smooth; (N+3)^3 extended
// elements, FDM cost ~12E(N+3)^4, ASM with the counting weight, RAS).
// oracle/schwarz.py states the algorithm on the CPU.
//
//   nk_fdm           one element per CTA, (N+3)^2 / 2 threads, each owning
//                    two 1-D lines of the extended box in shared memory:
//                    gather r (- sub) on the element and the face-neighbour
//                    layers -> S_x^T, S_y^T along lines -> (S_z^T, 1/Lambda,
//                    S_z) fused in one pass -> S_y, S_x -> extended (ASM) or
//                    own-point (RAS) output.  The 1-D S are per element
//                    (deformed meshes) and read broadcast from shared memory.
//                    6 (N+3)^4 DFMA per element, 2 (N+3)^3 shared transposes.
//   nk_schwarz_post  z = mask * W * (own points of the extended / own
//                    output) fused with the Chebyshev vector update
//                    d = a d + b z, e (+)= d.
#include <type_traits>

#include "common.cuh"

namespace nk {

__device__ __forceinline__ void fdm_dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// One thread's 1-D contractions of TWO lines L0, L1 (stride ST) in place:
//   L[a] = sum_i M[a][i] L[i]   (M rows of length SP in shared memory),
// optionally scaled by 1 / (lam0 (lab + lz[a]) + lam1) (0 when that sum is
// +inf: dropped points).  M is S^T for the forward and S for the backward
// transform.  Every M element loaded (16-B broadcast loads, all lanes on one
// address) feeds two FMAs (one per line): 1 shared load per 4 DFMA.
// 16-byte row chunks: 2 doubles or 4 floats per shared load
template <typename T> struct RowVec;
template <> struct RowVec<double> { static constexpr int W = 2; };
template <> struct RowVec<float> { static constexpr int W = 4; };
template <typename T> struct alignas(16) Chunk { T v[RowVec<T>::W]; };
template <int NQE, typename T>
struct RowPitch { static constexpr int SP = (NQE + RowVec<T>::W - 1) / RowVec<T>::W * RowVec<T>::W; };
__device__ __forceinline__ double fdm_rcp(double x) { return __drcp_rn(x); }
__device__ __forceinline__ float fdm_rcp(float x) { return __frcp_rn(x); }

template <int NQE, int ST, typename T>
__device__ __forceinline__ void fdm_line2(T* L0, T* L1, const T* __restrict__ M, const T* lz,
                                          T lab0, T lab1, T lam0, T lam1) {
  constexpr int W = RowVec<T>::W;
  constexpr int SP = RowPitch<NQE, T>::SP;
  T v0[NQE], v1[NQE];
#pragma unroll
  for (int i = 0; i < NQE; ++i) {
    v0[i] = L0[i * ST];
    v1[i] = L1[i * ST];
  }
#pragma unroll 2
  for (int a = 0; a < NQE; ++a) {
    const T* row = M + a * SP;
    T s0 = 0, s1 = 0;
#pragma unroll
    for (int i = 0; i + W <= NQE; i += W) {
      const Chunk<T> m = *reinterpret_cast<const Chunk<T>*>(row + i);
#pragma unroll
      for (int c = 0; c < W; ++c) {
        s0 = fma(m.v[c], v0[i + c], s0);
        s1 = fma(m.v[c], v1[i + c], s1);
      }
    }
#pragma unroll
    for (int i = NQE - NQE % W; i < NQE; ++i) {
      const T m = row[i];
      s0 = fma(m, v0[i], s0);
      s1 = fma(m, v1[i], s1);
    }
    if (lz != nullptr) {
      const T l0 = lab0 + lz[a], l1 = lab1 + lz[a];
      s0 = isinf(l0) ? T(0) : s0 * fdm_rcp(fma(lam0, l0, lam1));
      s1 = isinf(l1) ? T(0) : s1 * fdm_rcp(fma(lam0, l1, lam1));
    }
    L0[a * ST] = s0;
    L1[a * ST] = s1;
  }
}

template <int NQE, typename T>
struct FdmShape {
  static constexpr int NQ = NQE - 2;                 // N + 1
  static constexpr int LS = NQE + 1;                 // padded line stride
  static constexpr int PS = NQE * LS;                // plane stride
  static constexpr int SP = RowPitch<NQE, T>::SP;    // matrix row stride (16-B rows)
  static constexpr int NL = NQE * NQE;               // lines per orientation
  static constexpr int NT = (NL + 1) / 2;            // threads: two lines each
  static constexpr int A_SZ = (NQE * PS + RowVec<T>::W - 1) / RowVec<T>::W * RowVec<T>::W;  // 16-B aligned end
  static constexpr int M_SZ = 3 * NQE * SP;          // one of S^T / S, 3 directions
  static constexpr size_t SMEM = sizeof(T) * (A_SZ + 2 * M_SZ + 3 * NQE);
};

// One element per CTA, (N+3)^2 / 2 threads, two 1-D lines per thread and
// orientation, transposes through one padded shared box.
// T = double, or float for the 32-bit smoothing mode ("FP32
// is used only for the smoothing steps"): fields stay FP64 in HBM, the
// extended box, S and the spectrum are T in shared memory.
template <int NQE, typename T>
__global__ void __launch_bounds__(FdmShape<NQE, T>::NT)
fdm_kernel(int64_t nelem, const double* __restrict__ r, const double* __restrict__ sub,
           const double* __restrict__ rx, double* __restrict__ res_out,
           const int32_t* __restrict__ fmap,
           const T* __restrict__ Sg, const T* __restrict__ lamg, double lam0_d,
           double lam1_d, double* __restrict__ out, int out_ext, const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  using F = FdmShape<NQE, T>;
  const T lam0 = (T)lam0_d, lam1 = (T)lam1_d;
  constexpr int NQ = F::NQ;
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  constexpr int LS = F::LS, PS = F::PS, SP = F::SP, NT = F::NT, NL = F::NL;
  extern __shared__ __align__(16) unsigned char fdm_smem_raw[];
  T* A = reinterpret_cast<T*>(fdm_smem_raw);   // [k][j][i], padded lines
  T* Sf = A + F::A_SZ;                   // Sf[d][a][i] = S[d][i][a]  (forward)
  T* Sb = Sf + F::M_SZ;                  // Sb[d][i][a] = S[d][i][a]  (backward)
  T* Ls = Sb + F::M_SZ;                  // lambda[d][mode]
  const int64_t e = blockIdx.x;
  const int t = threadIdx.x;
  const T* Se = Sg + e * 3 * NQE * NQE;
  const int64_t ob = e * NQ3;
  const int32_t* fm = fmap + e * 6 * NQ2;
  // Global loads are issued in batches of CH independent loads per thread
  // (the gather is latency-bound: one element per CTA, few warps per SM).
  constexpr int CH = 8;
  constexpr int NS = 3 * NQE * NQE, NF = 6 * NQ2;
  for (int q0 = 0; q0 < NS; q0 += CH * NT) {
    T v[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      v[u] = q < NS ? __ldg(Se + q) : T(0);
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      if (q < NS) {
        const int d = q / (NQE * NQE), ia = q % (NQE * NQE), i = ia / NQE, a = ia % NQE;
        Sb[d * NQE * SP + i * SP + a] = v[u];
        Sf[d * NQE * SP + a * SP + i] = v[u];
      }
    }
  }
  for (int q = t; q < 3 * NQE; q += NT) Ls[q] = __ldg(lamg + e * 3 * NQE + q);
  for (int q = t; q < F::A_SZ; q += NT) A[q] = T(0);   // whole padded box, no index math
  __syncthreads();
  // own points (coalesced); res_out = r - sub on them
  for (int q0 = 0; q0 < NQ3; q0 += CH * NT) {
    double v[CH], w[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      v[u] = q < NQ3 ? __ldg(r + ob + q) : 0.0;
      w[u] = (sub != nullptr && q < NQ3) ? __ldg(sub + ob + q) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      if (q < NQ3) {
        const int i = q % NQ, j = (q / NQ) % NQ, k = q / NQ2;
        const double x = v[u] - w[u];
        if (res_out) res_out[ob + q] = x;
        A[(k + 1) * PS + (j + 1) * LS + (i + 1)] = (T)x;
      }
    }
  }
  // face-neighbour layers: face f, tangential (a, b) slow/fast
  for (int q0 = 0; q0 < NF; q0 += CH * NT) {
    int32_t src[CH];
    double v[CH], w[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      src[u] = q < NF ? __ldg(fm + q) : -1;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      // src >= 0: local point of r (- sub); src <= -2: a value received from
      // the neighbour rank (already r - sub) at rx[-src - 2]; -1: none
      v[u] = src[u] >= 0 ? __ldg(r + src[u]) : (src[u] <= -2 ? __ldg(rx - src[u] - 2) : 0.0);
      w[u] = (sub != nullptr && src[u] >= 0) ? __ldg(sub + src[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      if (src[u] != -1) {
        const int f = q / NQ2, ab = q % NQ2, a = ab / NQ + 1, b = ab % NQ + 1;
        const int pos = (f & 1) ? NQE - 1 : 0;
        int idx;
        if (f < 2) idx = a * PS + b * LS + pos;        // x faces: (k, j)
        else if (f < 4) idx = a * PS + pos * LS + b;   // y faces: (k, i)
        else idx = pos * PS + a * LS + b;              // z faces: (j, i)
        A[idx] = (T)(v[u] - w[u]);
      }
    }
  }
  __syncthreads();
  // this thread's two lines (the second clamped onto the first when NL is odd)
  const int l0 = t, l1 = (t + NT < NL) ? t + NT : t;
  const int h0 = l0 / NQE, o0 = l0 % NQE, h1 = l1 / NQE, o1 = l1 % NQE;
  constexpr int MD = NQE * SP;
  // forward x: lines (k = h, j = o) along i
  fdm_line2<NQE, 1, T>(A + h0 * PS + o0 * LS, A + h1 * PS + o1 * LS, Sf, nullptr, 0, 0, 0, 0);
  __syncthreads();
  // forward y: lines (k = h, i = o) along j
  fdm_line2<NQE, LS, T>(A + h0 * PS + o0, A + h1 * PS + o1, Sf + MD, nullptr, 0, 0, 0, 0);
  __syncthreads();
  // z: forward + inverse Kronecker-sum spectrum, then backward
  // (lines j = h -> mode b, i = o -> mode a, along k)
  fdm_line2<NQE, PS, T>(A + h0 * LS + o0, A + h1 * LS + o1, Sf + 2 * MD, Ls + 2 * NQE,
                     Ls[o0] + Ls[NQE + h0], Ls[o1] + Ls[NQE + h1], lam0, lam1);
  fdm_line2<NQE, PS, T>(A + h0 * LS + o0, A + h1 * LS + o1, Sb + 2 * MD, nullptr, 0, 0, 0, 0);
  __syncthreads();
  // backward y, backward x
  fdm_line2<NQE, LS, T>(A + h0 * PS + o0, A + h1 * PS + o1, Sb + MD, nullptr, 0, 0, 0, 0);
  __syncthreads();
  fdm_line2<NQE, 1, T>(A + h0 * PS + o0 * LS, A + h1 * PS + o1 * LS, Sb, nullptr, 0, 0, 0, 0);
  __syncthreads();
  if (out_ext) {
    // extended rows (k, j): NQE contiguous values each
    double* o = out + e * NQE * NQE * NQE;
    for (int rw = t; rw < NQE * NQE; rw += NT) {
      const T* srow = A + (rw / NQE) * PS + (rw % NQE) * LS;
#pragma unroll
      for (int i = 0; i < NQE; ++i) o[rw * NQE + i] = (double)srow[i];
    }
  } else {
    for (int q = t; q < NQ3; q += NT) {
      const int i = q % NQ, j = (q / NQ) % NQ, k = q / NQ2;
      out[ob + q] = (double)A[(k + 1) * PS + (j + 1) * LS + (i + 1)];
    }
  }
}

__global__ void __launch_bounds__(256)
schwarz_post_kernel(int nq, int64_t n, const double* __restrict__ src, int src_ext,
                    const double* __restrict__ W, const uint8_t* __restrict__ mask,
                    double* __restrict__ d, double* __restrict__ e, double a, double b,
                    int e_acc, const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int nq2 = nq * nq, nq3 = nq2 * nq, nqe = nq + 2, nqe2 = nqe * nqe;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    double z;
    if (src_ext) {
      const int64_t el = q / nq3;
      const int p = (int)(q - el * nq3);
      const int i = p % nq, j = (p / nq) % nq, k = p / nq2;
      z = __ldg(src + el * nqe2 * nqe + (int64_t)(k + 1) * nqe2 + (j + 1) * nqe + (i + 1));
    } else {
      z = __ldg(src + q);
    }
    if (W) z *= __ldg(W + q);
    if (mask && !mask[q]) z = 0.0;
    double dv = b * z;
    if (d) {
      if (a != 0.0) dv = fma(a, d[q], dv);
      d[q] = dv;
    }
    e[q] = e_acc ? e[q] + dv : dv;
  }
}


// ---------------------------------------------------------------------------
// nk_fdm on the FP64 tensor cores (NK_KNOB_FDM = 1, N + 3 <= 16).
//
// Why: the line kernel above is issue/latency-bound at ~24% of the FP64 rate
// (ncu r2o: short-scoreboard 31%, FP64 pipe 35%, ~0.45 shared-memory
// instructions per DFMA).  Each direction pass is the small GEMM
//   C[a][l] = sum_i M[a][i] B[i][l]   (M = S^T forward, S backward; B = the
//   box's (N+3)^2 lines along that direction)
// so a warp issues mma.sync.m8n8k4.f64 (SASS DMMA, 256 FMA per instruction)
// over 8-line tiles: A fragments (M, zero-padded to 16 x 4 KS) stay in
// registers for the pass, B fragments are one 8-byte shared load per lane
// and k-step, C goes back in place (the warp owns its tiles' lines for the
// pass; __syncwarp orders its reads before its writes).  The z pass applies
// the inverse Kronecker-sum spectrum to the C fragments and runs the backward
// z product on the same tile.  Padding (rows a >= N+3, k >= N+3, lines past
// (N+3)^2) is zero in A and predicated off in B / C.  Box layout: line stride
// LS and plane stride PS = 4 (mod 16) doubles, so one B-fragment load (4
// consecutive k of 8 lines) hits every bank exactly twice in the x and y
// passes.  4 warps per element (CTA).
template <int NQE>
struct FdmDmmaShape {
  static constexpr int NQ = NQE - 2;
  static constexpr int LS = NQE <= 4 ? 4 : 20;
  static constexpr int PS0 = NQE * LS;
  static constexpr int PS = PS0 + ((4 - PS0 % 16) + 16) % 16;
  static constexpr int KS = (NQE + 3) / 4, MT = (NQE + 7) / 8;
  static constexpr int NL = NQE * NQE, NTILE = (NL + 7) / 8;
  static constexpr int NW = 4, THREADS = 32 * NW;
  static constexpr int A_SZ = NQE * PS;
  // A | S | lambda | lab[NL] (x + y eigenvalue sum of each z line) | base[3][NL] (ints)
  static constexpr size_t SMEM =
      sizeof(double) * (A_SZ + 3 * NQE * NQE + 3 * NQE + NL) + sizeof(int) * 3 * NL;
};

template <int NQE>
__global__ void __launch_bounds__(FdmDmmaShape<NQE>::THREADS)
fdm_dmma_kernel(int64_t nelem, const double* __restrict__ r, const double* __restrict__ sub,
                const double* __restrict__ rx, double* __restrict__ res_out,
                const int32_t* __restrict__ fmap, const double* __restrict__ Sg,
                const double* __restrict__ lamg, double lam0, double lam1,
                double* __restrict__ out, int out_ext, const nk_cg_state* st) {
  static_assert(NQE <= 16, "two 8-row m tiles");
  if (st != nullptr && st->done) return;
  using F = FdmDmmaShape<NQE>;
  constexpr int NQ = F::NQ, NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  constexpr int LS = F::LS, PS = F::PS, KS = F::KS, MT = F::MT, NL = F::NL, NT = F::THREADS;
  extern __shared__ __align__(16) double fdm_dsmem[];
  double* A = fdm_dsmem;              // [k][j][i] at k*PS + j*LS + i
  double* Sm = A + F::A_SZ;           // S[d][i][a] as stored
  double* Ls = Sm + 3 * NQE * NQE;    // lambda[d][mode]
  double* lab = Ls + 3 * NQE;         // z line l = (j, i): lambda_x[i] + lambda_y[j]
  int* lbase = reinterpret_cast<int*>(lab + NL);   // [dir][line] -> A offset of k = 0
  const int64_t e = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, wq = t >> 5;
  const double* Se = Sg + e * 3 * NQE * NQE;
  const int64_t ob = e * NQ3;
  const int32_t* fm = fmap + e * 6 * NQ2;
  for (int q = t; q < 3 * NQE * NQE; q += NT) Sm[q] = __ldg(Se + q);
  for (int q = t; q < 3 * NQE; q += NT) Ls[q] = __ldg(lamg + e * 3 * NQE + q);
  for (int q = t; q < F::A_SZ; q += NT) A[q] = 0.0;
  for (int l = t; l < NL; l += NT) {
    const int h = l / NQE, o = l - h * NQE;
    lbase[l] = h * PS + o * LS;            // x lines (k = h, j = o) along i
    lbase[NL + l] = h * PS + o;            // y lines (k = h, i = o) along j
    lbase[2 * NL + l] = h * LS + o;        // z lines (j = h, i = o) along k
  }
  __syncthreads();
  for (int l = t; l < NL; l += NT) {
    const int h = l / NQE, o = l - h * NQE;
    lab[l] = Ls[o] + Ls[NQE + h];
  }
  constexpr int CH = 8;
  for (int q0 = 0; q0 < NQ3; q0 += CH * NT) {   // own points, res_out = r - sub
    double v[CH], w[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      v[u] = q < NQ3 ? __ldg(r + ob + q) : 0.0;
      w[u] = (sub != nullptr && q < NQ3) ? __ldg(sub + ob + q) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      if (q < NQ3) {
        const int i = q % NQ, j = (q / NQ) % NQ, k = q / NQ2;
        const double x = v[u] - w[u];
        if (res_out) res_out[ob + q] = x;
        A[(k + 1) * PS + (j + 1) * LS + (i + 1)] = x;
      }
    }
  }
  constexpr int NF = 6 * NQ2;
  for (int q0 = 0; q0 < NF; q0 += CH * NT) {    // face-neighbour layers (as fdm_kernel)
    int32_t src[CH];
    double v[CH], w[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      src[u] = q < NF ? __ldg(fm + q) : -1;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      v[u] = src[u] >= 0 ? __ldg(r + src[u]) : (src[u] <= -2 ? __ldg(rx - src[u] - 2) : 0.0);
      w[u] = (sub != nullptr && src[u] >= 0) ? __ldg(sub + src[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int q = q0 + u * NT + t;
      if (src[u] != -1) {
        const int f = q / NQ2, ab = q % NQ2, a = ab / NQ + 1, b = ab % NQ + 1;
        const int pos = (f & 1) ? NQE - 1 : 0;
        int idx;
        if (f < 2) idx = a * PS + b * LS + pos;
        else if (f < 4) idx = a * PS + pos * LS + b;
        else idx = pos * PS + a * LS + b;
        A[idx] = v[u] - w[u];
      }
    }
  }
  __syncthreads();

  auto base_of = [&](int dir, int l) -> int { return lbase[dir * NL + l]; };
  auto frags = [&](int dir, bool fwd, double (&af)[MT][KS]) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int a = mt * 8 + (lane >> 2), i = ks * 4 + (lane & 3);
        const double* S = Sm + dir * NQE * NQE;
        af[mt][ks] = (a < NQE && i < NQE) ? (fwd ? S[i * NQE + a] : S[a * NQE + i]) : 0.0;
      }
  };
  // one tile: C = M B over the tile's 8 lines (B read from A), optional
  // spectrum scaling, written back in place
  auto tile = [&](int dir, int st_, int nt, const double (&af)[MT][KS], bool scale) {
    const int lb = nt * 8 + (lane >> 2);
    const int bb = lb < NL ? base_of(dir, lb) : 0;
    double c[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) c[mt][0] = c[mt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int i = ks * 4 + (lane & 3);
      const double bv = (lb < NL && i < NQE) ? A[bb + i * st_] : 0.0;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) fdm_dmma884(c[mt][0], c[mt][1], af[mt][ks], bv);
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int a = mt * 8 + (lane >> 2), l = nt * 8 + 2 * (lane & 3) + hh;
        if (a < NQE && l < NL) {
          double val = c[mt][hh];
          if (scale) {
            const double l0 = lab[l] + Ls[2 * NQE + a];
            val = isinf(l0) ? 0.0 : val * fdm_rcp(fma(lam0, l0, lam1));
          }
          A[base_of(dir, l) + a * st_] = val;
        }
      }
    __syncwarp();
  };
  {
    double af[MT][KS];
    frags(0, true, af);   // forward x (along i)
    for (int nt = wq; nt < F::NTILE; nt += F::NW) tile(0, 1, nt, af, false);
    __syncthreads();
    frags(1, true, af);   // forward y (along j)
    for (int nt = wq; nt < F::NTILE; nt += F::NW) tile(1, LS, nt, af, false);
    __syncthreads();
    double ab[MT][KS];    // z: forward, spectrum, backward on the same tile
    frags(2, true, af);
    frags(2, false, ab);
    for (int nt = wq; nt < F::NTILE; nt += F::NW) {
      tile(2, PS, nt, af, true);
      tile(2, PS, nt, ab, false);
    }
    __syncthreads();
    frags(1, false, af);  // backward y, backward x
    for (int nt = wq; nt < F::NTILE; nt += F::NW) tile(1, LS, nt, af, false);
    __syncthreads();
    frags(0, false, af);
    for (int nt = wq; nt < F::NTILE; nt += F::NW) tile(0, 1, nt, af, false);
    __syncthreads();
  }
  if (out_ext) {
    double* o = out + e * NQE * NQE * NQE;
    for (int rw = t; rw < NQE * NQE; rw += NT) {
      const double* srow = A + (rw / NQE) * PS + (rw % NQE) * LS;
#pragma unroll
      for (int i = 0; i < NQE; ++i) o[rw * NQE + i] = srow[i];
    }
  } else {
    for (int q = t; q < NQ3; q += NT) {
      const int i = q % NQ, j = (q / NQ) % NQ, k = q / NQ2;
      out[ob + q] = A[(k + 1) * PS + (j + 1) * LS + (i + 1)];
    }
  }
}

template <int NQE, typename T>
static int launch_fdm(int64_t E, const double* r, const double* sub, const double* rx,
                      double* res_out,
                      const int32_t* fmap, const T* S, const T* lam, double lam0,
                      double lam1, double* out, int out_ext, const nk_cg_state* st,
                      cudaStream_t s) {
  if constexpr (std::is_same<T, double>::value && NQE <= 16) {
    // 2 = auto: the tensor-core path where it measured faster (scripts/prof_fdm.py
    // --fdm-knob, E = 16^3, profiles/r2zd_fdm_knob_sweep.jsonl): N + 3 a multiple
    // of 4 or >= 13 (1.05-1.62x); the 16 x 12 padding of the 10 x 10 operator
    // makes it lose at N = 7 (0.86x), and N <= 3 / 6 / 8 tie or lose
    const int kn = knob(NK_KNOB_FDM);
    const bool tc = kn == 1 || (kn == 2 && (NQE == 7 || NQE == 8 || NQE >= 12));
    if (tc) {
      constexpr size_t dsmem = FdmDmmaShape<NQE>::SMEM;
      static bool dconf = false;
      if (!dconf) {
        cudaError_t err = cudaFuncSetAttribute(fdm_dmma_kernel<NQE>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)dsmem);
        if (err != cudaSuccess) {
          set_error("fdm_dmma: smem attribute: %s", cudaGetErrorString(err));
          return NK_ERR_CUDA;
        }
        dconf = true;
      }
      fdm_dmma_kernel<NQE><<<(unsigned)E, FdmDmmaShape<NQE>::THREADS, dsmem, s>>>(
          E, r, sub, rx, res_out, fmap, S, lam, lam0, lam1, out, out_ext, st);
      return check_launch("fdm_dmma");
    }
  }
  constexpr size_t smem = FdmShape<NQE, T>::SMEM;
  static bool configured = false;
  if (!configured) {
    cudaError_t err = cudaFuncSetAttribute(fdm_kernel<NQE, T>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) {
      set_error("fdm: smem attribute: %s", cudaGetErrorString(err));
      return NK_ERR_CUDA;
    }
    configured = true;
  }
  fdm_kernel<NQE, T><<<(unsigned)E, FdmShape<NQE, T>::NT, smem, s>>>(E, r, sub, rx, res_out, fmap, S,
                                                                    lam, lam0, lam1, out, out_ext,
                                                                    st);
  return check_launch("fdm");
}

template <typename T>
static int fdm_dispatch(int N, int64_t nelem, const double* r, const double* sub,
                        const double* rx, double* res_out, const int32_t* fmap, const T* Smat, const T* lam,
                        double lam0, double lam1, double* out, int out_ext,
                        const nk_cg_state* st, nk_stream_t stream) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) {
    set_error("fdm: order %d outside [%d, %d]", N, NK_MIN_ORDER, NK_MAX_ORDER);
    return NK_ERR_UNSUPPORTED;
  }
  if (nelem < 0 || nelem > 0x7fffffffLL ||
      (nelem > 0 && (!r || !fmap || !Smat || !lam || !out))) {
    set_error("fdm: invalid arguments (nelem=%lld)", (long long)nelem);
    return NK_ERR_INVALID;
  }
  if (nelem == 0) return NK_OK;
  cudaStream_t s = S(stream);
  switch (N + 3) {
#define NK_FDM_CASE(Q) \
  case Q:              \
    return launch_fdm<Q, T>(nelem, r, sub, rx, res_out, fmap, Smat, lam, lam0, lam1, out, out_ext, \
                            st, s);
    NK_FDM_CASE(4) NK_FDM_CASE(5) NK_FDM_CASE(6) NK_FDM_CASE(7) NK_FDM_CASE(8) NK_FDM_CASE(9)
    NK_FDM_CASE(10) NK_FDM_CASE(11) NK_FDM_CASE(12) NK_FDM_CASE(13) NK_FDM_CASE(14)
    NK_FDM_CASE(15) NK_FDM_CASE(16) NK_FDM_CASE(17) NK_FDM_CASE(18)
#undef NK_FDM_CASE
    default: break;
  }
  set_error("fdm: order %d not instantiated", N);
  return NK_ERR_UNSUPPORTED;
}

}  // namespace nk

using namespace nk;

extern "C" int nk_fdm(int N, int64_t nelem, const double* r, const double* sub,
                      const double* rx, double* res_out, const int32_t* fmap, const double* Smat,
                      const double* lam, double lam0, double lam1, double* out, int out_ext,
                      const nk_cg_state* st, nk_stream_t stream) {
  return fdm_dispatch<double>(N, nelem, r, sub, rx, res_out, fmap, Smat, lam, lam0, lam1, out,
                              out_ext, st, stream);
}

extern "C" int nk_fdm32(int N, int64_t nelem, const double* r, const double* sub,
                        const double* rx, double* res_out, const int32_t* fmap,
                        const float* Smat, const float* lam, double lam0, double lam1,
                        double* out, int out_ext, const nk_cg_state* st, nk_stream_t stream) {
  return fdm_dispatch<float>(N, nelem, r, sub, rx, res_out, fmap, Smat, lam, lam0, lam1, out,
                             out_ext, st, stream);
}

// out[i] = a[idx[i]] - b[idx[i]] (b nullable): packs the face-inward layer
// values r - A e a neighbour rank's extended boxes need.
__global__ void __launch_bounds__(256)
gather_diff_kernel(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ a,
                   const double* __restrict__ b, double* __restrict__ out,
                   const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t q = __ldg(idx + i);
    out[i] = b ? __ldg(a + q) - __ldg(b + q) : __ldg(a + q);
  }
}

extern "C" int nk_gather_diff(int64_t n, const int32_t* idx, const double* a, const double* b,
                              double* out, const nk_cg_state* st, nk_stream_t stream) {
  if (n < 0 || (n > 0 && (!idx || !a || !out))) {
    set_error("gather_diff: invalid arguments");
    return NK_ERR_INVALID;
  }
  if (n == 0) return NK_OK;
  int64_t g = (n + 255) / 256;
  if (g > 8 * 148) g = 8 * 148;
  gather_diff_kernel<<<(unsigned)g, 256, 0, S(stream)>>>(n, idx, a, b, out, st);
  return check_launch("gather_diff");
}

extern "C" int nk_schwarz_post(int N, int64_t nelem, const double* src, int src_ext,
                               const double* W, const uint8_t* mask, double* d, double* e,
                               double a, double b, int e_acc, const nk_cg_state* st,
                               nk_stream_t stream) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER || nelem < 0 || (nelem > 0 && (!src || !e))) {
    set_error("schwarz_post: invalid arguments (N=%d nelem=%lld)", N, (long long)nelem);
    return NK_ERR_INVALID;
  }
  const int nq = N + 1;
  const int64_t n = nelem * nq * nq * nq;
  if (n == 0) return NK_OK;
  int64_t g = (n + 255) / 256;
  if (g > 8 * 148) g = 8 * 148;
  schwarz_post_kernel<<<(unsigned)g, 256, 0, S(stream)>>>(nq, n, src, src_ext, W, mask, d, e, a,
                                                          b, e_acc, st);
  return check_launch("schwarz_post");
}
