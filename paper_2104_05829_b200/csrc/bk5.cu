// BK5 dispatch by order (the kernels are in bk5_kernels.cuh, instantiated
// per order in bk5_inst.cu).
#include "common.cuh"

typedef int (*kslab_fn)(int, int64_t, const int32_t*, const double*, const double*, const double*,
                        double*, double, const double*, double, int64_t, const uint8_t*,
                        nk_cg_state*, double*, int64_t, int64_t, cudaStream_t, int64_t*, int,
                        int, int, int64_t);
typedef int (*diag_fn)(int64_t, const double*, const double*, double, const double*, double,
                       double*, cudaStream_t);

#define NK_DECL(NQ)                                                                          \
  extern "C" int nk_bk5_kslab_nq##NQ(int, int64_t, const int32_t*, const double*,            \
                                     const double*, const double*, double*, double,           \
                                     const double*, double, int64_t, const uint8_t*,          \
                                     nk_cg_state*, double*, int64_t, int64_t, cudaStream_t,   \
                                     int64_t*, int, int, int, int64_t);                       \
  extern "C" int nk_local_diag_nq##NQ(int64_t, const double*, const double*, double,         \
                                      const double*, double, double*, cudaStream_t);
#define NK_DECLP(NQ)                                                                        \
  extern "C" int nk_bk5_pcg_nq##NQ(int64_t, const int32_t*, const double*, const double*,  \
                                   double*, double*, double, const double*, double,          \
                                   const uint8_t*, double*, const double*, const double*,    \
                                   nk_cg_state*, double*, int64_t, int64_t, double*,          \
                                   cudaStream_t, int64_t*);
NK_DECLP(2) NK_DECLP(3) NK_DECLP(4) NK_DECLP(5) NK_DECLP(6) NK_DECLP(7) NK_DECLP(8) NK_DECLP(9)
NK_DECLP(10) NK_DECLP(11) NK_DECLP(12) NK_DECLP(13) NK_DECLP(14) NK_DECLP(15) NK_DECLP(16)
typedef int (*pcg_fn)(int64_t, const int32_t*, const double*, const double*, double*, double*,
                      double, const double*, double, const uint8_t*, double*, const double*,
                      const double*, nk_cg_state*, double*, int64_t, int64_t, double*,
                      cudaStream_t, int64_t*);
static const pcg_fn pcg_table[16] = {
    nullptr,          nk_bk5_pcg_nq2,  nk_bk5_pcg_nq3,  nk_bk5_pcg_nq4,  nk_bk5_pcg_nq5,
    nk_bk5_pcg_nq6,   nk_bk5_pcg_nq7,  nk_bk5_pcg_nq8,  nk_bk5_pcg_nq9,  nk_bk5_pcg_nq10,
    nk_bk5_pcg_nq11,  nk_bk5_pcg_nq12, nk_bk5_pcg_nq13, nk_bk5_pcg_nq14, nk_bk5_pcg_nq15,
    nk_bk5_pcg_nq16};

NK_DECL(2) NK_DECL(3) NK_DECL(4) NK_DECL(5) NK_DECL(6) NK_DECL(7) NK_DECL(8) NK_DECL(9)
NK_DECL(10) NK_DECL(11) NK_DECL(12) NK_DECL(13) NK_DECL(14) NK_DECL(15) NK_DECL(16)

static const kslab_fn kslab_table[16] = {
    nullptr,            nk_bk5_kslab_nq2,  nk_bk5_kslab_nq3,  nk_bk5_kslab_nq4,
    nk_bk5_kslab_nq5,   nk_bk5_kslab_nq6,  nk_bk5_kslab_nq7,  nk_bk5_kslab_nq8,
    nk_bk5_kslab_nq9,   nk_bk5_kslab_nq10, nk_bk5_kslab_nq11, nk_bk5_kslab_nq12,
    nk_bk5_kslab_nq13,  nk_bk5_kslab_nq14, nk_bk5_kslab_nq15, nk_bk5_kslab_nq16};
static const diag_fn diag_table[16] = {
    nullptr,              nk_local_diag_nq2,  nk_local_diag_nq3,  nk_local_diag_nq4,
    nk_local_diag_nq5,    nk_local_diag_nq6,  nk_local_diag_nq7,  nk_local_diag_nq8,
    nk_local_diag_nq9,    nk_local_diag_nq10, nk_local_diag_nq11, nk_local_diag_nq12,
    nk_local_diag_nq13,   nk_local_diag_nq14, nk_local_diag_nq15, nk_local_diag_nq16};

using namespace nk;

// tuning knobs (nk_bk5_tune): kslab shape index (N=7 only) and L2 prefetch
// distance in blocks (-1 = one wave, 0 = off)
static int g_cfg = 0;
static int g_pf = 1;

extern "C" int nk_bk5_tune(int cfg, int pf_dist) {
#ifndef NK_BK5_SHAPE_SWEEP
  if (cfg >= 11 && cfg <= 14) {
    set_error("bk5_tune: CTA-shape sweep configs 11..14 need a sweep build (make SWEEP=1)");
    return NK_ERR_UNSUPPORTED;
  }
#endif
  g_cfg = cfg;
  g_pf = pf_dist;
  return NK_OK;
}
extern "C" int nk_bk5_variant_get();

// auto (0): the measured winner per order (the select_kernel_variant of
// SPEC.md:420-428, decided offline by scripts/bk5_sweep.py --orders on the
// B200 under the cold-and-clean L2 protocol, profiles/r1_bk5_order_sweep*):
// pencil2 (2 shared buffers) where its extra residency wins, pencil
// elsewhere.  The fused BP5 step keeps its TMA pipeline (nk_bk5_pcg).
static int kvariant_for(int N) {
  const int v = nk_bk5_variant_get();
  if (v == 1 || v == 3 || v == 4 || v == 5) return v;
  if (v == 7) return N >= 8 ? 7 : 3;   // dmma: N + 1 >= 9
  if (v == 8) return (N >= 2 && N != 3) ? 8 : 3;   // stage: N + 1 in 3, 5..16
  if (v == 9) return (N >= 8 && N <= 14) ? 9 : 3;   // stage2: N + 1 in 9..15
  if (v == 10) return N == 15 ? 10 : 3;             // pair: N + 1 = 16
  if (v == 11) return N == 2 ? 11 : 3;              // point: N + 1 = 3
  switch (N) {   // measured: profiles/r2s_bk5_order_sweep_evenodd.jsonl, r2x_stage_sweep.jsonl,
                 // r2ze_stage_low.jsonl
    case 2: return 5;                                                        // pencil2
    case 6: case 8: case 9: case 10: case 12: case 13: case 14: case 15: return 8;   // stage
    default: return 3;                                      // pencil
  }
}

extern "C" int64_t nk_bk5_blocks(int N, int64_t nlist, int ncomp) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) return -1;
  int64_t nb = -1;
  kslab_table[N](ncomp, nlist, nullptr, nullptr, nullptr, nullptr, nullptr, 1.0, nullptr, 0.0, 0,
                 nullptr, nullptr, nullptr, 0, 0, nullptr, &nb, g_cfg, g_pf, kvariant_for(N), 0);
  return nb;
}

// the 3-component kernel the auto table picks per order (-1: three scalar
// launches), measured on the B200 (scripts/bk5_sweep.py --helm3,
// profiles/r2zg_helm3.jsonl, re-measured after the stage kernel):
//   seq3    -- bk5_pencil<NC = 3>: the three components back to back in one
//              CTA, G from HBM once and re-read from L2 (N = 3, 5, 7..13);
//   pencil3 -- the three components interleaved, G in registers once
//              (N = 4, 6);
//   scalar  -- three scalar launches of the auto kernel (N = 1, 2, 14, 15).
// (pencil3 also edges out seq3 at N = 7 and 9, by 3-8%; seq3 is kept there
// because the batched PCG's fused per-component dots need it.)
// A forced variant (nk_bk5_set_variant) keeps its own kernel: 6 = seq3,
// any other = pencil3 / k-slab.
static int helm3_variant(int N) {
  int v = nk_bk5_variant_get();
  if (v != 0) return v;
  switch (N) {
    case 3: case 5: case 7: case 8: case 9: case 10: case 11: case 12: case 13: return 6;
    case 4: case 6: return 3;
    default: return -1;
  }
}

extern "C" int64_t nk_bk5_batch_blocks(int N, int64_t nlist) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) return -1;
  int64_t nb = -1;
  const int v = helm3_variant(N);
  if (v == 6)
    kslab_table[N](3, nlist, nullptr, nullptr, nullptr, nullptr, nullptr, 1.0, nullptr, 0.0, 0,
                   nullptr, nullptr, nullptr, 0, 0, nullptr, &nb, g_cfg, g_pf, 6, 0);
  else
    kslab_table[N](1, nlist, nullptr, nullptr, nullptr, nullptr, nullptr, 1.0, nullptr, 0.0, 0,
                   nullptr, nullptr, nullptr, 0, 0, nullptr, &nb, g_cfg, g_pf, kvariant_for(N), 0);
  return nb;
}

extern "C" int nk_bk5_batch_variant(int N) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) return -2;
  return helm3_variant(N);
}

extern "C" int nk_bk5(int N, int64_t nelem, const double* D, const double* G, const double* u,
                      double* w, double lam0, const double* B, double lam1, int ncomp,
                      int64_t comp_stride, const uint8_t* mask, const int32_t* elem_list,
                      int64_t nlist, nk_cg_state* st, double* partials, int64_t part_base,
                      int64_t reduce_count, nk_stream_t stream) {
  if (ncomp == 3 && st != nullptr) {
    set_error("bk5: the fused dots of a 3-component batch need nk_bk5_batch");
    return NK_ERR_INVALID;
  }
  return nk_bk5_batch(N, nelem, D, G, u, w, lam0, B, lam1, ncomp, comp_stride, mask, elem_list,
                      nlist, st, partials, 0, part_base, reduce_count, stream);
}

extern "C" int nk_bk5_batch(int N, int64_t nelem, const double* D, const double* G,
                            const double* u, double* w, double lam0, const double* B,
                            double lam1, int ncomp, int64_t comp_stride, const uint8_t* mask,
                            const int32_t* elem_list, int64_t nlist, nk_cg_state* st,
                            double* partials, int64_t part_stride, int64_t part_base,
                            int64_t reduce_count, nk_stream_t stream) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) {
    set_error("bk5: order N=%d outside compiled range [%d, %d]", N, NK_MIN_ORDER, NK_MAX_ORDER);
    return NK_ERR_UNSUPPORTED;
  }
  if (ncomp != 1 && ncomp != 3) {
    set_error("bk5: ncomp must be 1 or 3 (got %d)", ncomp);
    return NK_ERR_INVALID;
  }
  if (!D || !G || !u || !w || nelem < 0) {
    set_error("bk5: null operand");
    return NK_ERR_INVALID;
  }
  if (B == nullptr && lam1 != 0.0) {
    set_error("bk5: lam1 != 0 requires B");
    return NK_ERR_INVALID;
  }
  if (st != nullptr && partials == nullptr) {
    set_error("bk5: fused dot needs partials");
    return NK_ERR_INVALID;
  }
  const int64_t n = elem_list ? nlist : nelem;
  if (ncomp > 1 && comp_stride < nelem * (int64_t)(N + 1) * (N + 1) * (N + 1)) {
    set_error("bk5: comp_stride too small");
    return NK_ERR_INVALID;
  }
  if (ncomp > 1 && st != nullptr && part_stride < (reduce_count > 0 ? reduce_count : 1)) {
    set_error("bk5: part_stride too small for the per-component partials");
    return NK_ERR_INVALID;
  }
  cudaStream_t s = S(stream);
  const int64_t nq3 = (int64_t)(N + 1) * (N + 1) * (N + 1);
  if (ncomp == 3) {
    int v = helm3_variant(N);
    // fused per-component dots: seq3 or three scalar launches
    if (st != nullptr && v != 6) v = -1;
    if (v == -1) {
      for (int c = 0; c < 3; ++c) {
        int rc = kslab_table[N](1, n, elem_list, D, G, u + c * comp_stride, w + c * comp_stride,
                                lam0, B, lam1, nelem * nq3, mask, st ? st + c : nullptr,
                                st ? partials + c * part_stride : nullptr, part_base,
                                reduce_count, s, nullptr, g_cfg, g_pf, kvariant_for(N), 0);
        if (rc != NK_OK) return rc;
      }
      return NK_OK;
    }
    return kslab_table[N](3, n, elem_list, D, G, u, w, lam0, B, lam1, comp_stride, mask, st,
                          partials, part_base, reduce_count, s, nullptr, g_cfg, g_pf, v,
                          part_stride);
  }
  // ncomp = 1: the stride slot carries the u array length (nelem NQ^3
  // doubles), which bounds the 16-byte rounded bulk copies of bk5_stage
  return kslab_table[N](ncomp, n, elem_list, D, G, u, w, lam0, B, lam1, nelem * nq3, mask, st,
                        partials, part_base, reduce_count, s, nullptr, g_cfg, g_pf,
                        kvariant_for(N), 0);
}

extern "C" int nk_local_diag(int N, int64_t nelem, const double* D, const double* G, double lam0,
                             const double* B, double lam1, double* diag, nk_stream_t stream) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) {
    set_error("local_diag: order N=%d unsupported", N);
    return NK_ERR_UNSUPPORTED;
  }
  if (!D || !G || !diag) {
    set_error("local_diag: null operand");
    return NK_ERR_INVALID;
  }
  return diag_table[N](nelem, D, G, lam0, B, lam1, diag, S(stream));
}

extern "C" int64_t nk_bk5_pcg_blocks(int N, int64_t nlist) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) return -1;
  int64_t nb = -1;
  pcg_table[N](nlist, nullptr, nullptr, nullptr, nullptr, nullptr, 1.0, nullptr, 0.0, nullptr,
               nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, nullptr, nullptr, &nb);
  return nb;
}

extern "C" int nk_bk5_pcg(int N, int64_t nelem, const double* D, const double* G, double* p,
                          double* w, double lam0, const double* B, double lam1,
                          const uint8_t* mask, const int32_t* elem_list, int64_t nlist,
                          double* x, const double* r, const double* invD, nk_cg_state* st,
                          double* partials, int64_t part_base, int64_t reduce_count,
                          double* hist, nk_stream_t stream) {
  if (N < NK_MIN_ORDER || N > NK_MAX_ORDER) {
    set_error("bk5_pcg: order N=%d outside compiled range", N);
    return NK_ERR_UNSUPPORTED;
  }
  if (!D || !G || !p || !w || !x || !r || !invD || !st || !partials || nelem < 0) {
    set_error("bk5_pcg: null operand");
    return NK_ERR_INVALID;
  }
  if (B == nullptr && lam1 != 0.0) {
    set_error("bk5_pcg: lam1 != 0 requires B");
    return NK_ERR_INVALID;
  }
  const int64_t n = elem_list ? nlist : nelem;
  return pcg_table[N](n, elem_list, D, G, p, w, lam0, B, lam1, mask, x, r, invD, st, partials,
                      part_base, reduce_count, hist, S(stream), nullptr);
}

// ---------------------------------------------- the step + edge/vertex gs
extern "C" int nk_bk5_pcg_gs_fused(int N) {
  return (knob(NK_KNOB_GS_TAIL) == 1 && N == 7 && nk_bk5_variant_get() != 3) ? 1 : 0;
}

extern "C" int nk_bk5_pcg_gs(int N, int64_t nelem, const double* D, const double* G, double* p,
                             double* w, double lam0, const double* B, double lam1,
                             const uint8_t* mask, double* x, const double* r,
                             const double* invD, nk_cg_state* st, double* partials,
                             int64_t reduce_count, double* hist, int nclass,
                             const int32_t* sizes, const int64_t* nsegs,
                             const int32_t* const* members, nk_stream_t stream) {
  GsTail T{};
  const int rcb = gs_tail_build(T, nclass, sizes, nsegs, members);
  if (rcb != NK_OK) return rcb;
  const int k = T.n;
  const bool offer = k > 0 && nk_bk5_pcg_gs_fused(N);
  gs_tail_set(offer ? &T : nullptr);
  const int rc = nk_bk5_pcg(N, nelem, D, G, p, w, lam0, B, lam1, mask, nullptr, 0, x, r, invD, st,
                            partials, 0, reduce_count, hist, stream);
  const bool used = offer && gs_tail_used();
  gs_tail_set(nullptr);
  if (rc != NK_OK || used || k == 0) return rc;
  return nk_gs_op_classes(nclass, sizes, nsegs, members, w, NK_OP_ADD, 1, 0, st, stream);
}
