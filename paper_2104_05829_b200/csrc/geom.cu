// Device-side mesh setup for generated boxes:
// coordinates (trilinear then deformed), geometric factors from dx/dr = D_q x
// (PAPER.md:1177-1180, 1213-1218, 1256-1263), lattice global ids and the
// Dirichlet mask.  Setup only -- runs once per mesh -- but on device so the
// 134M-point configurations do not spend minutes in host numpy.
#include <climits>

#include <cuda.h>

#include "common.cuh"

namespace nk {

struct BoxDesc {
  int32_t nx, ny, nz;
  double ex, ey, ez;   // extent
  double ox, oy, oz;   // origin
};

__device__ __forceinline__ void elem_xyz(int64_t e, const BoxDesc& b, int64_t* ex, int64_t* ey,
                                         int64_t* ez) {
  *ex = e % b.nx;
  *ey = (e / b.nx) % b.ny;
  *ez = e / ((int64_t)b.nx * b.ny);
}

__global__ void box_coords_kernel(int N, int64_t nelem, const int64_t* __restrict__ eidx,
                                  BoxDesc b, int deform, double amp,
                                  const double* __restrict__ nodes, double* __restrict__ xyz) {
  const int nq = N + 1;
  const int64_t nq3 = (int64_t)nq * nq * nq;
  const int64_t n = nelem * nq3;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t le = p / nq3;
  const int r = (int)(p - le * nq3);
  const int i = r % nq, j = (r / nq) % nq, k = r / (nq * nq);
  const int64_t e = eidx ? eidx[le] : le;
  int64_t ex, ey, ez;
  elem_xyz(e, b, &ex, &ey, &ez);
  const double hx = b.ex / b.nx, hy = b.ey / b.ny, hz = b.ez / b.nz;
  double x = b.ox + ((double)ex + 0.5 * (nodes[i] + 1.0)) * hx;
  double y = b.oy + ((double)ey + 0.5 * (nodes[j] + 1.0)) * hy;
  double z = b.oz + ((double)ez + 0.5 * (nodes[k] + 1.0)) * hz;
  if (deform == NK_DEFORM_SINE) {
    const double X = (x - b.ox) / b.ex, Y = (y - b.oy) / b.ey, Z = (z - b.oz) / b.ez;
    const double pi = 3.141592653589793;
    const double sx = sin(pi * X), sy = sin(pi * Y), sz = sin(pi * Z);
    const double dx = amp * b.ex * sin(2 * pi * X) * sy * sz;
    const double dy = amp * b.ey * sx * sin(2 * pi * Y) * sz;
    const double dz = amp * b.ez * sx * sy * sin(2 * pi * Z);
    x += dx;
    y += dy;
    z += dz;
  }
  xyz[p] = x;
  xyz[n + p] = y;
  xyz[2 * n + p] = z;
}

// one thread per point; derivatives read coordinates straight from global
// (L1-resident within an element).
__global__ void geom_factors_kernel(int N, int64_t nelem, const double* __restrict__ D,
                                    const double* __restrict__ wts,
                                    const double* __restrict__ xyz, double* __restrict__ G,
                                    double* __restrict__ B, double* __restrict__ Jout,
                                    double* __restrict__ rxout, int64_t* status) {
  const int nq = N + 1;
  const int64_t nq2 = (int64_t)nq * nq, nq3 = nq2 * nq;
  const int64_t n = nelem * nq3;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t e = p / nq3;
  const int r = (int)(p - e * nq3);
  const int i = r % nq, j = (r / nq) % nq, k = r / (nq * nq);
  double a[3][3];  // a[c][q] = dx_c / dr_q
  for (int c = 0; c < 3; ++c) {
    const double* X = xyz + c * n + e * nq3;
    double dr = 0.0, ds = 0.0, dt = 0.0;
    for (int m = 0; m < nq; ++m) {
      dr += D[i * nq + m] * X[k * nq2 + j * nq + m];
      ds += D[j * nq + m] * X[k * nq2 + m * nq + i];
      dt += D[k * nq + m] * X[m * nq2 + j * nq + i];
    }
    a[c][0] = dr;
    a[c][1] = ds;
    a[c][2] = dt;
  }
  const double J = a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
                   a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
                   a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
  if (fabs(J) < 1e-14) atomicMin((unsigned long long*)&status[0], (unsigned long long)e);
  if (J <= 0.0) atomicMin((unsigned long long*)&status[1], (unsigned long long)e);
  // rx[q][c] = dr_q/dx_c = cofactor(c,q)/J
  double rx[3][3];
  for (int c = 0; c < 3; ++c)
    for (int q = 0; q < 3; ++q) {
      const int c1 = (c + 1) % 3, c2 = (c + 2) % 3, q1 = (q + 1) % 3, q2 = (q + 2) % 3;
      rx[q][c] = (a[c1][q1] * a[c2][q2] - a[c1][q2] * a[c2][q1]) / J;
    }
  const double wJ = wts[i] * wts[j] * wts[k] * J;
  const int pairs[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
  double* Ge = G + e * 6 * nq3 + r;
  for (int q = 0; q < 6; ++q) {
    const int m = pairs[q][0], mm = pairs[q][1];
    Ge[q * nq3] = (rx[m][0] * rx[mm][0] + rx[m][1] * rx[mm][1] + rx[m][2] * rx[mm][2]) * wJ;
  }
  B[p] = wJ;
  if (Jout) Jout[p] = J;
  if (rxout)
    for (int q = 0; q < 3; ++q)
      for (int c = 0; c < 3; ++c) rxout[(q * 3 + c) * n + p] = rx[q][c];
}

__global__ void box_ids_kernel(int N, int64_t nelem, const int64_t* __restrict__ eidx, BoxDesc b,
                               int px, int py, int pz, int64_t* __restrict__ ids) {
  const int nq = N + 1;
  const int64_t nq3 = (int64_t)nq * nq * nq;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nelem * nq3) return;
  const int64_t le = p / nq3;
  const int r = (int)(p - le * nq3);
  const int i = r % nq, j = (r / nq) % nq, k = r / (nq * nq);
  const int64_t e = eidx ? eidx[le] : le;
  int64_t ex, ey, ez;
  elem_xyz(e, b, &ex, &ey, &ez);
  const int64_t Lx = (int64_t)b.nx * N, Ly = (int64_t)b.ny * N, Lz = (int64_t)b.nz * N;
  int64_t gx = ex * N + i, gy = ey * N + j, gz = ez * N + k;
  int64_t sx = Lx + 1, sy = Ly + 1;
  if (px) { gx %= Lx; sx = Lx; }
  if (py) { gy %= Ly; sy = Ly; }
  if (pz) { gz %= Lz; }
  ids[p] = (gz * sy + gy) * sx + gx + 1;
}

__global__ void box_mask_kernel(int N, int64_t nelem, const int64_t* __restrict__ eidx, BoxDesc b,
                                int dm, uint8_t* __restrict__ mask) {
  const int nq = N + 1;
  const int64_t nq3 = (int64_t)nq * nq * nq;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nelem * nq3) return;
  const int64_t le = p / nq3;
  const int r = (int)(p - le * nq3);
  const int i = r % nq, j = (r / nq) % nq, k = r / (nq * nq);
  const int64_t e = eidx ? eidx[le] : le;
  int64_t ex, ey, ez;
  elem_xyz(e, b, &ex, &ey, &ez);
  bool zero = ((dm & 1) && ex == 0 && i == 0) || ((dm & 2) && ex == b.nx - 1 && i == N) ||
              ((dm & 4) && ey == 0 && j == 0) || ((dm & 8) && ey == b.ny - 1 && j == N) ||
              ((dm & 16) && ez == 0 && k == 0) || ((dm & 32) && ez == b.nz - 1 && k == N);
  mask[p] = zero ? 0 : 1;
}

__global__ void l2_flush_kernel(int4* buf, int64_t n16, int v) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n16; q += stride)
    buf[q] = make_int4(v, v, v, v);
}

// Read-only sweep: evicts the (dirty) lines the write sweep left in L2, so
// the next timed kernel starts with a cold AND clean L2 (no write-backs of
// flush data charged to it).
__global__ void l2_clean_kernel(const int4* __restrict__ buf, int64_t n16, int* sink) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int acc = 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n16; q += stride) {
    const int4 v = __ldcg(buf + q);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x7fffffff) *sink = acc;  // keep the loads alive
}

// Bandwidth probe with BK5's exact HBM pattern: per element read u (nq3) and
// G (6 nq3), write w (nq3) -- no arithmetic beyond a sum.  The achievable
// ceiling for the BK5 byte mix, measured the same way as BK5.
__global__ void __launch_bounds__(256) bw_probe_kernel(int64_t npts, int nq3,
                                                       const double2* __restrict__ u,
                                                       const double2* __restrict__ G,
                                                       double2* __restrict__ w) {
  const int64_t n2 = npts / 2;
  const int h = nq3 / 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += stride) {
    const int64_t e = q / h, r = q - e * h;
    double2 acc = __ldg(u + q);
    const double2* g = G + e * 6 * h + r;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const double2 v = __ldg(g + c * h);
      acc.x += v.x;
      acc.y += v.y;
    }
    w[q] = acc;
  }
}

static BoxDesc make_desc(const int32_t* counts, const double* extent, const double* origin) {
  BoxDesc d;
  d.nx = counts[0];
  d.ny = counts[1];
  d.nz = counts[2];
  d.ex = extent ? extent[0] : 1.0;
  d.ey = extent ? extent[1] : 1.0;
  d.ez = extent ? extent[2] : 1.0;
  d.ox = origin ? origin[0] : 0.0;
  d.oy = origin ? origin[1] : 0.0;
  d.oz = origin ? origin[2] : 0.0;
  return d;
}

static unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace nk

using namespace nk;

static bool bad_counts(const int32_t* c) { return !c || c[0] < 1 || c[1] < 1 || c[2] < 1; }

extern "C" int nk_box_coords(int N, int64_t nelem, const int64_t* elem_index,
                             const int32_t* counts, const double* extent, const double* origin,
                             int deform_kind, double amp, const double* nodes, double* xyz,
                             nk_stream_t stream) {
  if (N < 1 || nelem < 0 || bad_counts(counts) || !extent || !nodes || !xyz) {
    set_error("box_coords: invalid arguments");
    return NK_ERR_INVALID;
  }
  if (deform_kind != NK_DEFORM_NONE && deform_kind != NK_DEFORM_SINE) {
    set_error("box_coords: unknown deformation %d", deform_kind);
    return NK_ERR_INVALID;
  }
  const int64_t n = nelem * (int64_t)(N + 1) * (N + 1) * (N + 1);
  if (n == 0) return NK_OK;
  box_coords_kernel<<<blocks_for(n), 256, 0, S(stream)>>>(
      N, nelem, elem_index, make_desc(counts, extent, origin), deform_kind, amp, nodes, xyz);
  return check_launch("box_coords");
}

extern "C" int nk_geom_factors(int N, int64_t nelem, const double* D, const double* weights,
                               const double* xyz, double* G, double* B, double* J,
                               double* rx, int64_t* status, nk_stream_t stream) {
  if (N < 1 || nelem < 0 || !D || !weights || !xyz || !G || !B || !status) {
    set_error("geom_factors: invalid arguments");
    return NK_ERR_INVALID;
  }
  const int64_t n = nelem * (int64_t)(N + 1) * (N + 1) * (N + 1);
  if (n == 0) return NK_OK;
  geom_factors_kernel<<<blocks_for(n), 256, 0, S(stream)>>>(N, nelem, D, weights, xyz, G, B, J,
                                                            rx, status);
  return check_launch("geom_factors");
}

extern "C" int nk_box_ids(int N, int64_t nelem, const int64_t* elem_index, const int32_t* counts,
                          const int32_t* periodic, int64_t* ids, nk_stream_t stream) {
  if (N < 1 || nelem < 0 || bad_counts(counts) || !ids) {
    set_error("box_ids: invalid arguments");
    return NK_ERR_INVALID;
  }
  const int64_t n = nelem * (int64_t)(N + 1) * (N + 1) * (N + 1);
  if (n == 0) return NK_OK;
  const int px = periodic ? periodic[0] : 0, py = periodic ? periodic[1] : 0,
            pz = periodic ? periodic[2] : 0;
  box_ids_kernel<<<blocks_for(n), 256, 0, S(stream)>>>(
      N, nelem, elem_index, make_desc(counts, nullptr, nullptr), px, py, pz, ids);
  return check_launch("box_ids");
}

extern "C" int nk_box_mask(int N, int64_t nelem, const int64_t* elem_index, const int32_t* counts,
                           const int32_t* dirichlet, uint8_t* mask, nk_stream_t stream) {
  if (N < 1 || nelem < 0 || bad_counts(counts) || !dirichlet || !mask) {
    set_error("box_mask: invalid arguments");
    return NK_ERR_INVALID;
  }
  int dm = 0;
  for (int f = 0; f < 6; ++f)
    if (dirichlet[f]) dm |= 1 << f;
  const int64_t n = nelem * (int64_t)(N + 1) * (N + 1) * (N + 1);
  if (n == 0) return NK_OK;
  box_mask_kernel<<<blocks_for(n), 256, 0, S(stream)>>>(
      N, nelem, elem_index, make_desc(counts, nullptr, nullptr), dm, mask);
  return check_launch("box_mask");
}

extern "C" int nk_bw_probe(int64_t nelem, int nq3, const double* u, const double* G, double* w,
                           int blocks_per_sm, nk_stream_t stream) {
  if (nelem < 0 || nq3 % 2 || !u || !G || !w) {
    set_error("bw_probe: invalid arguments");
    return NK_ERR_INVALID;
  }
  const int bps = blocks_per_sm > 0 ? blocks_per_sm : 8;
  bw_probe_kernel<<<148 * bps, 256, 0, S(stream)>>>(nelem * nq3, nq3, (const double2*)u,
                                                     (const double2*)G, (double2*)w);
  return check_launch("bw_probe");
}

extern "C" int nk_l2_flush(void* buf, int64_t bytes, nk_stream_t stream) {
  if (!buf || bytes < 16) {
    set_error("l2_flush: buffer too small");
    return NK_ERR_INVALID;
  }
  static int v = 0;
  ++v;
  // first half: write sweep (flush); second half: read sweep (clean)
  const int64_t half16 = bytes / 32;
  l2_flush_kernel<<<148 * 8, 256, 0, S(stream)>>>((int4*)buf, half16, v);
  int rc = check_launch("l2_flush");
  if (rc) return rc;
  int4* second = (int4*)buf + half16;
  l2_clean_kernel<<<148 * 8, 256, 0, S(stream)>>>(second, half16, (int*)buf);
  return check_launch("l2_clean");
}

// Stream-ordered 64-bit write by the GPU front end (cuStreamWriteValue64: no
// copy engine, no SM), ordered after all prior work of the stream; capturable
// into CUDA graphs (memory-operation node).  The chunk gate of the streamed
// host-buffer BK5 (nk_bk5_set_gate).
extern "C" int nk_stream_write_u64(void* dptr, uint64_t value, nk_stream_t stream) {
  typedef CUresult (*Fn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
  static Fn fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", reinterpret_cast<void**>(&fn),
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr) {
      fn = nullptr;
      set_error("stream_write_u64: cuStreamWriteValue64 unavailable");
      return NK_ERR_CUDA;
    }
  }
  if (!dptr) {
    set_error("stream_write_u64: null pointer");
    return NK_ERR_INVALID;
  }
  const CUresult r = fn(reinterpret_cast<CUstream>(S(stream)),
                        reinterpret_cast<CUdeviceptr>(dptr), value, 0);
  if (r != CUDA_SUCCESS) {
    set_error("stream_write_u64: cuStreamWriteValue64 failed (%d)", (int)r);
    return NK_ERR_CUDA;
  }
  return NK_OK;
}
