// One translation unit per order (compiled with -DNK_BK5_NQ=N+1) so the
// heavily unrolled BK5 instantiations build in parallel.
#include "bk5_kernels.cuh"

#ifndef NK_BK5_NQ
#error "compile with -DNK_BK5_NQ=<N+1>"
#endif
#define NK_CAT2(a, b) a##b
#define NK_CAT(a, b) NK_CAT2(a, b)

using namespace nk;

extern "C" int NK_CAT(nk_bk5_kslab_nq, NK_BK5_NQ)(int ncomp, int64_t nlist, const int32_t* elist,
                                                 const double* D, const double* G, const double* u,
                                                 double* w, double lam0, const double* B,
                                                 double lam1, int64_t cstride, const uint8_t* mask,
                                                 nk_cg_state* st, double* partials,
                                                 int64_t part_base, int64_t reduce_count,
                                                 cudaStream_t s, int64_t* nblocks) {
  constexpr int NQ = NK_BK5_NQ;
  if (nblocks) {
    *nblocks = kslab_blocks<NQ>(nlist);
    return NK_OK;
  }
  if (ncomp == 1)
    return launch_kslab<NQ, 1>(nlist, elist, D, G, u, w, lam0, B, lam1, cstride, mask, st,
                               partials, part_base, reduce_count, s);
  return launch_kslab<NQ, 3>(nlist, elist, D, G, u, w, lam0, B, lam1, cstride, mask, st,
                             partials, part_base, reduce_count, s);
}

extern "C" int NK_CAT(nk_local_diag_nq, NK_BK5_NQ)(int64_t nelem, const double* D,
                                                  const double* G, double lam0, const double* B,
                                                  double lam1, double* diag, cudaStream_t s) {
  constexpr int NQ = NK_BK5_NQ;
  const int64_t n = nelem * NQ * NQ * NQ;
  if (n == 0) return NK_OK;
  local_diag_kernel<NQ><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nelem, D, G, lam0, B, lam1,
                                                                     diag);
  return check_launch("local_diag");
}
