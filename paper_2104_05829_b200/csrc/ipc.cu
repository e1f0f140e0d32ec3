// NCCL-free halo transport over NVLink peer memory (CUDA IPC mappings).
//
// gs_op_overlapped's exchange step done
// by kernels instead of a collective: the pack kernel stores every boundary
// contribution directly into the neighbour GPU's receive buffer (remote
// st.global over NVLink/NVSwitch), and its last block publishes a per-pair
// epoch flag with a system-scope release; the combine kernel acquire-waits
// on the flags of all neighbours and folds the contributions in canonical
// order.  Receive buffers are double-buffered by epoch parity: a peer can
// run at most one exchange ahead (its next combine waits for our next push,
// which stream-order follows our current combine), so parity slots never
// collide.  Epochs live in device memory so the exchange can be replayed
// inside a CUDA graph.
#include <cstring>

#include "common.cuh"

namespace nk {

struct HaloPeers {
  int n;                        // neighbours
  double* recv[8];              // peer receive buffer base (mapped)
  int64_t recv_off[8];          // where our contributions start in the peer's buffer
  int64_t recv_len[8];          // peer buffer length (parity stride)
  unsigned long long* flag[8];  // peer flag word for our pair (mapped)
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// epoch[0]: exchanges completed by this rank (incremented by the push's last
// block); epoch[1]: last-block ticket.
__global__ void halo_push_kernel(const __grid_constant__ HaloPeers P,
                                 const int32_t* __restrict__ send_start,
                                 const int32_t* __restrict__ send_idx,
                                 const double* __restrict__ w, unsigned long long* epoch,
                                 const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const unsigned long long ep = epoch[0] + 1;     // the exchange being performed
  const int par = (int)(ep & 1);
  const int64_t total = send_start[P.n];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += stride) {
    int q = 0;
    while (q + 1 < P.n && g >= send_start[q + 1]) ++q;
    const int64_t i = g - send_start[q];
    P.recv[q][par * P.recv_len[q] + P.recv_off[q] + i] = w[send_idx[g]];
  }
  __threadfence_system();
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(reinterpret_cast<unsigned*>(epoch + 1), 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    epoch[1] = 0;
    epoch[0] = ep;
    for (int q = 0; q < P.n; ++q) st_release_sys(P.flag[q], ep);
  }
}

// combine with the wait folded in: every block acquires all neighbour flags
// (>= this rank's current epoch) before reading the receive buffer.
template <int OP>
__global__ void halo_combine_wait_kernel(int64_t nh, const int32_t* __restrict__ src_start,
                                         const int32_t* __restrict__ src_idx,
                                         const double* __restrict__ buf, int64_t buf_len,
                                         int64_t own_len, const int32_t* __restrict__ dst_start,
                                         const int32_t* __restrict__ dst_idx,
                                         double* __restrict__ w, const unsigned long long* flags,
                                         int nflags, const unsigned long long* epoch,
                                         const nk_cg_state* st) {
  if (st != nullptr && st->done) return;
  const unsigned long long ep = *(volatile const unsigned long long*)epoch;
  if (threadIdx.x < nflags) {
    while (ld_acquire_sys(flags + threadIdx.x) < ep) {
    }
  }
  __syncthreads();
  const int par = (int)(ep & 1);
  const double* rb = buf + par * buf_len;   // received part of this parity
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += stride) {
    const int a = src_start[h], b = src_start[h + 1];
    auto val = [&](int s) -> double {
      // own contributions live in the non-parity region [0, own_len) of the
      // parity-0 copy; received ones in the current parity's copy
      return s < own_len ? buf[s] : rb[s];
    };
    double acc = val(src_idx[a]);
    for (int q = a + 1; q < b; ++q) {
      const double v = val(src_idx[q]);
      if (OP == NK_OP_ADD) acc += v;
      else if (OP == NK_OP_MUL) acc *= v;
      else if (OP == NK_OP_MIN) acc = fmin(acc, v);
      else acc = fmax(acc, v);
    }
    for (int q = dst_start[h]; q < dst_start[h + 1]; ++q) w[dst_idx[q]] = acc;
  }
}

}  // namespace nk

using namespace nk;

extern "C" int nk_ipc_alloc(int64_t bytes, void** ptr, void* handle) {
  if (bytes <= 0 || !ptr || !handle) {
    set_error("ipc_alloc: invalid arguments");
    return NK_ERR_INVALID;
  }
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, (size_t)bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle((cudaIpcMemHandle_t*)handle, *ptr);
  if (e != cudaSuccess) {
    set_error("ipc_alloc: %s", cudaGetErrorString(e));
    return NK_ERR_CUDA;
  }
  return NK_OK;
}

extern "C" int nk_ipc_free(void* ptr) {
  if (ptr) cudaFree(ptr);
  return NK_OK;
}

extern "C" int nk_ipc_open(const void* handle, void** peer_ptr) {
  if (!handle || !peer_ptr) {
    set_error("ipc_open: invalid arguments");
    return NK_ERR_INVALID;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(peer_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error("ipc_open: %s", cudaGetErrorString(e));
    return NK_ERR_CUDA;
  }
  return NK_OK;
}

extern "C" int nk_ipc_close(void* peer_ptr) {
  if (peer_ptr) cudaIpcCloseMemHandle(peer_ptr);
  return NK_OK;
}

extern "C" int nk_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

extern "C" int nk_halo_push(int nnb, void* const* peer_recv, const int64_t* recv_off,
                            const int64_t* recv_len, void* const* peer_flag,
                            const int32_t* send_start, const int32_t* send_idx, const double* w,
                            int64_t total, uint64_t* epoch, const nk_cg_state* st,
                            nk_stream_t stream) {
  if (nnb < 0 || nnb > 8 || (nnb > 0 && (!peer_recv || !recv_off || !recv_len || !peer_flag)) ||
      !epoch) {
    set_error("halo_push: invalid arguments (at most 8 neighbours)");
    return NK_ERR_INVALID;
  }
  HaloPeers P{};
  P.n = nnb;
  for (int q = 0; q < nnb; ++q) {
    P.recv[q] = (double*)peer_recv[q];
    P.recv_off[q] = recv_off[q];
    P.recv_len[q] = recv_len[q];
    P.flag[q] = (unsigned long long*)peer_flag[q];
  }
  int64_t g = (total + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 4) g = 148 * 4;
  halo_push_kernel<<<(unsigned)g, 256, 0, S(stream)>>>(P, send_start, send_idx, w,
                                                      (unsigned long long*)epoch, st);
  return check_launch("halo_push");
}

extern "C" int nk_halo_combine_wait(int64_t nh, const int32_t* src_start, const int32_t* src_idx,
                                    const double* buf, int64_t buf_len, int64_t own_len,
                                    const int32_t* dst_start, const int32_t* dst_idx, double* w,
                                    int op, const uint64_t* flags, int nflags,
                                    const uint64_t* epoch, const nk_cg_state* st,
                                    nk_stream_t stream) {
  if (nh == 0) return NK_OK;
  if (nflags > 1024 || !buf || !epoch || (nflags > 0 && !flags)) {
    set_error("halo_combine_wait: invalid arguments");
    return NK_ERR_INVALID;
  }
  int64_t g = (nh + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  cudaStream_t s = S(stream);
  const auto* F = (const unsigned long long*)flags;
  const auto* E = (const unsigned long long*)epoch;
  switch (op) {
    case NK_OP_ADD: halo_combine_wait_kernel<NK_OP_ADD><<<(unsigned)g, 256, 0, s>>>(nh, src_start, src_idx, buf, buf_len, own_len, dst_start, dst_idx, w, F, nflags, E, st); break;
    case NK_OP_MUL: halo_combine_wait_kernel<NK_OP_MUL><<<(unsigned)g, 256, 0, s>>>(nh, src_start, src_idx, buf, buf_len, own_len, dst_start, dst_idx, w, F, nflags, E, st); break;
    case NK_OP_MIN: halo_combine_wait_kernel<NK_OP_MIN><<<(unsigned)g, 256, 0, s>>>(nh, src_start, src_idx, buf, buf_len, own_len, dst_start, dst_idx, w, F, nflags, E, st); break;
    case NK_OP_MAX: halo_combine_wait_kernel<NK_OP_MAX><<<(unsigned)g, 256, 0, s>>>(nh, src_start, src_idx, buf, buf_len, own_len, dst_start, dst_idx, w, F, nflags, E, st); break;
    default: set_error("halo_combine_wait: unknown op %d", op); return NK_ERR_INVALID;
  }
  return check_launch("halo_combine_wait");
}

// ---------------------------------------------------------------------------
// Scalar all-reduce over peer memory ("board"): every rank writes its k <= 4
// partial sums into slot [parity][rank] of every rank's board (own included)
// and releases a per-writer flag; the reduce kernel acquire-waits on all
// nranks flags and sums the slots in rank order -- deterministic and
// bitwise identical on every rank, graph-replayable (epochs in device
// memory), no NCCL.  Parity double-buffering: a rank's push e+1 follows its
// reduce e, which needed everyone's push e, so at most one epoch of skew.
namespace nk {

struct BoardPeers {
  int n, rank, k;
  double* board[8];              // each rank's board base (own included)
  unsigned long long* flag[8];   // flag word for THIS rank inside each board owner
};

__global__ void board_push_kernel(const __grid_constant__ BoardPeers P, const double* vals,
                                  unsigned long long* epoch) {
  const unsigned long long ep = epoch[0] + 1;
  const int par = (int)(ep & 1);
  const int q = threadIdx.x;
  if (q < P.n) {
    double* dst = P.board[q] + ((size_t)par * P.n + P.rank) * 4;
    for (int j = 0; j < P.k; ++j) dst[j] = vals[j];
    __threadfence_system();
    st_release_sys(P.flag[q], ep);
  }
  __syncthreads();
  if (q == 0) epoch[0] = ep;
}

__global__ void board_reduce_kernel(int n, int k, const double* board,
                                    const unsigned long long* flags,
                                    const unsigned long long* epoch, double* dst) {
  const unsigned long long ep = *(volatile const unsigned long long*)epoch;
  if (threadIdx.x < n) {
    while (ld_acquire_sys(flags + threadIdx.x) < ep) {
    }
  }
  __syncthreads();
  if (threadIdx.x < k) {
    const int par = (int)(ep & 1);
    double s = 0.0;
    for (int r = 0; r < n; ++r) s += board[((size_t)par * n + r) * 4 + threadIdx.x];
    dst[threadIdx.x] = s;
  }
}

}  // namespace nk

extern "C" int nk_board_allreduce(int nranks, int rank, double* vals, int k,
                                  void* const* boards, void* const* flags_for_me,
                                  const double* my_board, const uint64_t* my_flags,
                                  uint64_t* epoch, nk_stream_t stream) {
  if (nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks || k < 1 || k > 4 || !vals ||
      !boards || !flags_for_me || !my_board || !my_flags || !epoch) {
    set_error("board_allreduce: invalid arguments (<= 8 ranks, k <= 4)");
    return NK_ERR_INVALID;
  }
  BoardPeers P{};
  P.n = nranks;
  P.rank = rank;
  P.k = k;
  for (int q = 0; q < nranks; ++q) {
    P.board[q] = (double*)boards[q];
    P.flag[q] = (unsigned long long*)flags_for_me[q];
  }
  cudaStream_t s = S(stream);
  board_push_kernel<<<1, 32, 0, s>>>(P, vals, (unsigned long long*)epoch);
  int rc = check_launch("board_push");
  if (rc) return rc;
  board_reduce_kernel<<<1, 32, 0, s>>>(nranks, k, my_board, (const unsigned long long*)my_flags,
                                       (const unsigned long long*)epoch, vals);
  return check_launch("board_reduce");
}
