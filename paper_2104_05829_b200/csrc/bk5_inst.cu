// One translation unit per order (compiled with -DNK_BK5_NQ=N+1) so the
// heavily unrolled BK5 instantiations build in parallel.
#include "bk5_tma.cuh"
#include "bk5_pcg.cuh"
#include "bk5_pencil3.cuh"
#include "bk5_dmma.cuh"
#include "bk5_stage.cuh"
#include "bk5_stage2.cuh"
#include "bk5_pair.cuh"
#include "bk5_point.cuh"

#ifndef NK_BK5_NQ
#error "compile with -DNK_BK5_NQ=<N+1>"
#endif
#define NK_CAT2(a, b) a##b
#define NK_CAT(a, b) NK_CAT2(a, b)

using namespace nk;

extern "C" int nk_bk5_variant_get();

namespace {
// pf_dist < 0: one wave ahead (resident CTAs on the device), 0: off.
template <int NQ, int NC, int EPB, int MINB>
int run(int64_t nlist, const int32_t* elist, const double* D, const double* G, const double* u,
        double* w, double lam0, const double* B, double lam1, int64_t cstride,
        const uint8_t* mask, nk_cg_state* st, double* partials, int64_t part_base,
        int64_t reduce_count, cudaStream_t s, int64_t* nblocks, int pf_dist) {
  if (nblocks) {
    *nblocks = kslab_blocks<NQ, EPB>(nlist);
    return NK_OK;
  }
  if (pf_dist < 0) {
    static int wave = -1;
    if (wave < 0) {
      int dev = 0, sms = 148, per = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      using C = Bk5Cfg<NQ, EPB, MINB>;
      cudaFuncSetAttribute(bk5_kslab<NQ, NC, EPB, MINB>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes(NC));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk5_kslab<NQ, NC, EPB, MINB>,
                                                    C::THREADS, C::smem_bytes(NC));
      wave = sms * (per > 0 ? per : 1);
    }
    pf_dist = wave;
  }
  return launch_kslab<NQ, NC, EPB, MINB>(nlist, elist, D, G, u, w, lam0, B, lam1, cstride, mask,
                                         st, partials, part_base, reduce_count, s, pf_dist);
}

// Default shapes: one element per CTA; MINB from the order sweep
// (profiles/r1k_high_shapes.jsonl): at NQ >= 10 a lower MINB (higher register
// cap, no spills) beats the extra resident CTAs -- multi-element CTAs, which
// would pack NQ^2 threads into whole warps, spill and lose at every order.
template <int NQ> struct PencilDefault;
#define NK_PD(NQ_, EPB_, MINB_) \
  template <> struct PencilDefault<NQ_> { static constexpr int EPB = EPB_, MINB = MINB_; };
NK_PD(2, 32, 8) NK_PD(3, 14, 6) NK_PD(4, 4, 12) NK_PD(5, 5, 6) NK_PD(6, 2, 10) NK_PD(7, 2, 8)
NK_PD(8, 1, 10) NK_PD(9, 1, 8) NK_PD(10, 1, 5) NK_PD(11, 1, 4) NK_PD(12, 1, 3) NK_PD(13, 1, 2)
NK_PD(14, 1, 2) NK_PD(15, 1, 2) NK_PD(16, 1, 2)
#undef NK_PD

template <int NQ, int EPB, int MINB>
int runp(int64_t nlist, const int32_t* elist, const double* D, const double* G, const double* u,
         double* w, double lam0, const double* B, double lam1, const uint8_t* mask,
         nk_cg_state* st, double* partials, int64_t part_base, int64_t reduce_count,
         cudaStream_t s, int64_t* nblocks, int pfG) {
  if (nblocks) {
    *nblocks = pencil_dot_blocks<NQ, EPB, MINB>(nlist);
    return NK_OK;
  }
  return launch_pencil<NQ, EPB, MINB>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials,
                                      part_base, reduce_count, s, pfG);
}

// pencil2 shapes: 2 element buffers allow ~1.5x the resident CTAs of pencil
template <int NQ> struct Pencil2Default;
#define NK_P2D(NQ_, EPB_, MINB_) \
  template <> struct Pencil2Default<NQ_> { static constexpr int EPB = EPB_, MINB = MINB_; };
NK_P2D(2, 32, 8) NK_P2D(3, 14, 6) NK_P2D(4, 4, 14) NK_P2D(5, 5, 8) NK_P2D(6, 2, 12)
NK_P2D(7, 2, 5) NK_P2D(8, 1, 8) NK_P2D(9, 1, 5) NK_P2D(10, 1, 4) NK_P2D(11, 1, 4)
NK_P2D(12, 1, 3) NK_P2D(13, 1, 3) NK_P2D(14, 1, 2) NK_P2D(15, 1, 2) NK_P2D(16, 1, 2)
#undef NK_P2D


// Alternative (EPB, MINB) shapes for NQ >= 3 (not 8: own table), selected by nk_bk5_tune(cfg = 11..14)
// in a sweep build (make SWEEP=1 -> -DNK_BK5_SHAPE_SWEEP; the product build
// does not instantiate them)
// for the order sweep (scripts/bk5_sweep.py --high-shapes): several elements per
// CTA pack NQ^2-thread elements into whole warps (e.g. NQ = 13: 169 -> 192
// threads, 2 x 169 -> 352).
template <int NQ> struct PencilAlt {
  static constexpr int E[4] = {1, 1, 1, 1}, M[4] = {1, 1, 1, 1};
};
#define NK_ALT(NQ_, e0, m0, e1, m1, e2, m2, e3, m3)                 \
  template <> struct PencilAlt<NQ_> {                               \
    static constexpr int E[4] = {e0, e1, e2, e3}, M[4] = {m0, m1, m2, m3}; \
  };
NK_ALT(3, 32, 6, 28, 4, 14, 8, 7, 12) NK_ALT(4, 8, 6, 4, 16, 2, 16, 8, 8)
NK_ALT(5, 5, 8, 5, 4, 10, 3, 10, 4) NK_ALT(6, 8, 3, 8, 4, 4, 6, 7, 4)
NK_ALT(7, 1, 16, 2, 10, 5, 4, 4, 4)
NK_ALT(9, 1, 6, 1, 5, 1, 4, 1, 3) NK_ALT(10, 1, 5, 1, 4, 1, 3, 1, 2)
NK_ALT(11, 1, 4, 1, 3, 1, 2, 1, 1) NK_ALT(12, 1, 3, 1, 2, 1, 1, 2, 1)
NK_ALT(13, 1, 2, 1, 1, 2, 1, 1, 4) NK_ALT(14, 1, 2, 1, 1, 2, 1, 1, 4)
NK_ALT(15, 1, 1, 1, 3, 2, 1, 1, 4) NK_ALT(16, 1, 1, 2, 1, 1, 3, 1, 4)
#undef NK_ALT

template <int NQ>
int run_pencil2(int cfg, int64_t nlist, const int32_t* elist, const double* D, const double* G,
                const double* u, double* w, double lam0, const double* B, double lam1,
                const uint8_t* mask, nk_cg_state* st, double* partials, int64_t part_base,
                int64_t reduce_count, cudaStream_t s, int64_t* nb, int pfG) {
#ifdef NK_BK5_SHAPE_SWEEP
  if constexpr (NQ >= 3 && NQ != 8) {
    if (cfg >= 11 && cfg <= 14) {
      using A = PencilAlt<NQ>;
#define NK_P2ALT(K)                                                                           \
  if (cfg == 11 + K) {                                                                        \
    if (nb) {                                                                                 \
      *nb = pencil2_dot_blocks<NQ, A::E[K], A::M[K]>(nlist);                                   \
      return NK_OK;                                                                           \
    }                                                                                         \
    return launch_pencil2<NQ, A::E[K], A::M[K]>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, \
                                                st, partials, part_base, reduce_count, s, pfG); \
  }
      NK_P2ALT(0) NK_P2ALT(1) NK_P2ALT(2) NK_P2ALT(3)
#undef NK_P2ALT
    }
  }
#endif
  constexpr int EPB = Pencil2Default<NQ>::EPB, MINB = Pencil2Default<NQ>::MINB;
  if (nb) {
    *nb = pencil2_dot_blocks<NQ, EPB, MINB>(nlist);
    return NK_OK;
  }
  return launch_pencil2<NQ, EPB, MINB>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st,
                                       partials, part_base, reduce_count, s, pfG);
}

template <int NQ>
int run_pencil(int cfg, int64_t nlist, const int32_t* elist, const double* D, const double* G,
               const double* u, double* w, double lam0, const double* B, double lam1,
               const uint8_t* mask, nk_cg_state* st, double* partials, int64_t part_base,
               int64_t reduce_count, cudaStream_t s, int64_t* nb, int pfG) {
#define NK_PARGS nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base, \
                 reduce_count, s, nb, pfG
  if constexpr (NQ == 8) {
    switch (cfg) {
      case 1: return runp<8, 4, 4>(NK_PARGS);
      case 2: return runp<8, 2, 6>(NK_PARGS);
      case 3: return runp<8, 2, 8>(NK_PARGS);
      case 5: return runp<8, 4, 2>(NK_PARGS);
      case 6: return runp<8, 8, 1>(NK_PARGS);
      case 7: return runp<8, 4, 3>(NK_PARGS);
      case 8: return runp<8, 1, 12>(NK_PARGS);
      case 9: return runp<8, 1, 14>(NK_PARGS);
      default: return runp<8, 1, 10>(NK_PARGS);   // measured best (sweep16)
    }
  } else {
#ifdef NK_BK5_SHAPE_SWEEP
    if constexpr (NQ >= 3) {
      using A = PencilAlt<NQ>;
      switch (cfg) {
        case 11: return runp<NQ, A::E[0], A::M[0]>(NK_PARGS);
        case 12: return runp<NQ, A::E[1], A::M[1]>(NK_PARGS);
        case 13: return runp<NQ, A::E[2], A::M[2]>(NK_PARGS);
        case 14: return runp<NQ, A::E[3], A::M[3]>(NK_PARGS);
        default: break;
      }
    }
#endif
    return runp<NQ, PencilDefault<NQ>::EPB, PencilDefault<NQ>::MINB>(NK_PARGS);
  }
#undef NK_PARGS
}

template <int NQ, int MINB>
int runt(int64_t nlist, const int32_t* elist, const double* D, const double* G, const double* u,
         double* w, double lam0, const double* B, double lam1, const uint8_t* mask,
         nk_cg_state* st, double* partials, int64_t part_base, int64_t reduce_count,
         cudaStream_t s, int64_t* nblocks) {
  if (nblocks) {
    *nblocks = tma_grid<NQ, MINB>(nlist);
    return NK_OK;
  }
  return launch_pencil_tma<NQ, MINB>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials,
                                     part_base, reduce_count, s);
}

// bk5_stage (variant 8) shapes per order: NGS of the six G components staged
// in shared memory, NUB u buffers (2: u(next) issued an element ahead and w
// bulk-stored), MINB CTAs per SM.  cfg 0 is the default; nk_bk5_tune cfg 21 /
// 22 select two alternatives for the sweep (scripts/bk5_hot.py --sweep).
// U = 3: two u buffers with R in the current one (RINU, odd NQ); U = 4: two
// u buffers, G component NGS staged in the spare one (G4U).  E:
// elements per CTA (the low orders run several small elements side by side).
template <int NQ> struct StageShapes {
  static constexpr int G[3] = {6, 6, 6}, U[3] = {2, 1, 2}, M[3] = {1, 1, 1}, E[3] = {1, 1, 1};
};
#define NK_SDE(NQ_, g0, u0, m0, e0, g1, u1, m1, e1, g2, u2, m2, e2)                        \
  template <> struct StageShapes<NQ_> {                                                   \
    static constexpr int G[3] = {g0, g1, g2}, U[3] = {u0, u1, u2}, M[3] = {m0, m1, m2},   \
                         E[3] = {e0, e1, e2};                                             \
  };
#define NK_SD(NQ_, g0, u0, m0, g1, u1, m1, g2, u2, m2) \
  NK_SDE(NQ_, g0, u0, m0, 1, g1, u1, m1, 1, g2, u2, m2, 1)
NK_SDE(3, 6, 2, 4, 16, 6, 2, 2, 32, 6, 2, 8, 8) NK_SDE(5, 6, 2, 4, 5, 6, 2, 5, 4, 6, 2, 2, 8)
NK_SDE(6, 6, 2, 6, 2, 6, 2, 3, 4, 6, 2, 8, 1) NK_SDE(7, 6, 2, 4, 2, 6, 2, 2, 4, 6, 2, 6, 1)
NK_SD(8, 6, 2, 5, 6, 2, 4, 6, 2, 3) NK_SD(9, 6, 2, 3, 6, 2, 2, 6, 1, 3)
NK_SD(10, 6, 2, 2, 6, 1, 3, 4, 2, 3) NK_SD(11, 6, 2, 2, 4, 1, 3, 6, 2, 1)
NK_SD(12, 6, 2, 1, 4, 1, 3, 6, 2, 2) NK_SD(13, 6, 2, 1, 3, 2, 2, 6, 1, 1)
NK_SD(14, 6, 2, 1, 2, 2, 2, 6, 1, 1) NK_SD(15, 4, 2, 1, 5, 3, 1, 4, 4, 1)
#undef NK_SD
#undef NK_SDE

// bk5_stage2 (variant 9, two threads per pencil): (NGS, MINB) per order
template <int NQ> struct Stage2Shape { static constexpr int G = 6, M = 1; };
#define NK_S2(NQ_, g, m) \
  template <> struct Stage2Shape<NQ_> { static constexpr int G = g, M = m; };
NK_S2(9, 6, 2) NK_S2(10, 6, 2) NK_S2(11, 6, 2) NK_S2(12, 6, 1) NK_S2(13, 6, 1) NK_S2(14, 6, 1)
NK_S2(15, 4, 1)
#undef NK_S2

template <int NQ, int NGS, int NUB, int MINB, int EPB>
int runs(int64_t nlist, const int32_t* elist, const double* D, const double* G, const double* u,
         double* w, double lam0, const double* B, double lam1, const uint8_t* mask,
         nk_cg_state* st, double* partials, int64_t part_base, int64_t reduce_count,
         int64_t u_len, cudaStream_t s, int64_t* nblocks) {
  constexpr int NB = NUB >= 3 ? 2 : NUB;
  constexpr bool RINU = NUB == 3, G4U = NUB == 4;
  if (nblocks) {
    *nblocks = stage_grid<NQ, NGS, NB, MINB, RINU, EPB, G4U>(nlist);
    return NK_OK;
  }
  return launch_stage<NQ, NGS, NB, MINB, RINU, EPB, G4U>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials,
                                     part_base, reduce_count, u_len, s);
}

template <int NQ, int NC>
int run_cfg(int cfg, int64_t nlist, const int32_t* elist, const double* D, const double* G,
            const double* u, double* w, double lam0, const double* B, double lam1,
            int64_t cstride, const uint8_t* mask, nk_cg_state* st, double* partials,
            int64_t part_base, int64_t reduce_count, cudaStream_t s, int64_t* nb, int pf) {
#define NK_ARGS nlist, elist, D, G, u, w, lam0, B, lam1, cstride, mask, st, partials, part_base, \
                reduce_count, s, nb, pf
  if constexpr (NQ == 8 && NC == 1) {
    switch (cfg) {
      case 1: return run<NQ, NC, 4, 3>(NK_ARGS);
      case 2: return run<NQ, NC, 2, 4>(NK_ARGS);
      case 3: return run<NQ, NC, 2, 6>(NK_ARGS);
      case 4: return run<NQ, NC, 1, 8>(NK_ARGS);
      case 5: return run<NQ, NC, 1, 12>(NK_ARGS);
      case 6: return run<NQ, NC, 8, 1>(NK_ARGS);
      default: break;
    }
  }
  return run<NQ, NC, Bk5Cfg<NQ>::EPB, Bk5Cfg<NQ>::MINB>(NK_ARGS);
#undef NK_ARGS
}
}  // namespace

extern "C" int NK_CAT(nk_bk5_kslab_nq, NK_BK5_NQ)(int ncomp, int64_t nlist, const int32_t* elist,
                                                 const double* D, const double* G, const double* u,
                                                 double* w, double lam0, const double* B,
                                                 double lam1, int64_t cstride, const uint8_t* mask,
                                                 nk_cg_state* st, double* partials,
                                                 int64_t part_base, int64_t reduce_count,
                                                 cudaStream_t s, int64_t* nblocks, int cfg,
                                                 int pf_dist, int variant, int64_t pstride) {
  constexpr int NQ = NK_BK5_NQ;
  if constexpr (NQ == 2) {   // N = 1: element per thread unless k-slab is forced
    if (ncomp == 1 && variant != 1) {
      const int64_t nb = (nlist * 8 + kN1PtThreads - 1) / kN1PtThreads;
      const int64_t nbd = nb < kN1DotBlocks ? nb : kN1DotBlocks;   // fused dot: capped, looped
      if (nblocks) {
        *nblocks = nbd;
        return NK_OK;
      }
      if (nb == 0) return NK_OK;
      DParam<2> Dp;
      Dp.set(D);
      if (st != nullptr)
        bk5_n1<2, true><<<(unsigned)nbd, kN1PtThreads, 0, s>>>(
            nlist, elist, Dp, G, u, w, lam0, B, lam1, mask, st, partials, part_base, reduce_count);
      else
        bk5_n1<2><<<(unsigned)nb, kN1PtThreads, 0, s>>>(nlist, elist, Dp, G, u, w, lam0, B, lam1,
                                                      mask, st, partials, part_base, reduce_count);
      return check_launch("bk5_n1");
    }
  }
  if constexpr (NQ == 3) {
    // point per thread (bk5_point.cuh): whole-array calls with 16-byte
    // aligned u and G; element lists and other alignments take pencil2
    if (variant == 11 && ncomp == 1 && elist == nullptr &&
        ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(G)) & 15) == 0) {
      if (nblocks) {
        *nblocks = point3_blocks(nlist);
        return NK_OK;
      }
      return launch_point3(nlist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base,
                           reduce_count, s);
    }
    if (variant == 11) variant = 5;
  }
  if constexpr (NQ == 4 || NQ == 6 || NQ == 8) {
    if (variant == 4 && ncomp == 1) {
#define NK_TARGS nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base, \
                 reduce_count, s, nblocks
      if (NQ == 8 && cfg == 1) return runt<NQ, 2>(NK_TARGS);
      return runt<NQ, NQ == 8 ? 3 : (NQ == 6 ? 6 : 8)>(NK_TARGS);
#undef NK_TARGS
    }
  }
  if (ncomp == 3 && variant == 6) {
    // 3 components back to back per CTA, G from HBM once (bk5_pencil NC = 3);
    // with st: three CG states, per-component fused p.Ap (nk_bk5_batch)
#ifdef NK_BK5_SHAPE_SWEEP
    if constexpr (NQ >= 3 && NQ != 8) {
      using A = PencilAlt<NQ>;
#define NK_S3ALT(K)                                                                             \
  if (cfg == 11 + K) {                                                                          \
    if (nblocks) {                                                                              \
      *nblocks = (nlist + A::E[K] - 1) / A::E[K];                                               \
      return NK_OK;                                                                             \
    }                                                                                           \
    return launch_pencil<NQ, A::E[K], A::M[K], 3>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, \
                                                  nullptr, nullptr, 0, 0, s, pf_dist, cstride);  \
  }
      NK_S3ALT(0) NK_S3ALT(1) NK_S3ALT(2) NK_S3ALT(3)
#undef NK_S3ALT
    }
#endif
    // seq3 keeps the scalar shape except N = 9: one MINB lower (4, not 5)
    // drops its 96 B spill (profiles/r1l_seq3_shapes.jsonl)
    constexpr int EPB = PencilDefault<NQ>::EPB;
    constexpr int MINB = NQ == 10 ? 4 : PencilDefault<NQ>::MINB;
    if (nblocks) {
      *nblocks = (nlist + EPB - 1) / EPB;
      return NK_OK;
    }
    return launch_pencil<NQ, EPB, MINB, 3>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st,
                                           partials, part_base, reduce_count, s, pf_dist, cstride,
                                           pstride);
  }
  if constexpr (NQ >= 2 && NQ <= 12) {
    // 3-component batch: G read once per element (pencil3); k-slab otherwise
    if (ncomp == 3 && variant != 1) {
      if (nblocks) {
        *nblocks = nlist;
        return NK_OK;
      }
      if (st != nullptr) {
        set_error("bk5: the fused dot is not available for ncomp = 3");
        return NK_ERR_INVALID;
      }
      // smem 7 element buffers: NQ 8 -> 32 KB, 10 -> 57 KB, 12 -> 105 KB per CTA
      constexpr int M3 = NQ <= 6 ? 4 : (NQ <= 8 ? 3 : (NQ <= 10 ? 2 : 1));
      return launch_pencil3<NQ, M3>(nlist, elist, D, G, u, w, lam0, B, lam1, cstride, mask, s);
    }
  }
  if constexpr (NQ >= 9) {
    if (variant == 7 && ncomp == 1) {   // FP64 tensor-core contractions (bk5_dmma.cuh)
      constexpr int MINB = NQ <= 14 ? 2 : 1;   // shared memory fits two CTAs up to NQ = 14
      if (nblocks) {
        *nblocks = dmma_grid<NQ, MINB>(nlist);
        return NK_OK;
      }
      return launch_dmma<NQ, MINB>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials,
                                   part_base, reduce_count, s);
    }
  }
#if NK_BK5_NQ == 16
  if constexpr (NQ == 16) {
    if (variant == 10 && ncomp == 1) {   // one element per CTA pair (bk5_pair.cuh)
      if (nblocks) {
        *nblocks = pair16_grid(nlist);
        return NK_OK;
      }
      return launch_pair16(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials,
                           part_base, reduce_count, cstride, s);
    }
    if (variant == 8 && ncomp == 1) {   // tensor-map (swizzled) staging (bk5_stage.cuh)
      if (nblocks) {
        *nblocks = stage16_grid(nlist);
        return NK_OK;
      }
      // needs 16-byte aligned u, w, G (tensor maps); errors otherwise (the
      // pencil kernels' 16-byte row loads need the same at even NQ)
      return launch_stage16(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials,
                            part_base, reduce_count, cstride, s);
    }
  }
#endif
  if constexpr (NQ >= 9 && NQ <= 15) {
    if (variant == 9 && ncomp == 1) {   // stage with two threads per pencil (bk5_stage2.cuh)
      using S2 = Stage2Shape<NQ>;
      if (nblocks) {
        *nblocks = stage2_grid<NQ, S2::G, S2::M>(nlist);
        return NK_OK;
      }
      return launch_stage2<NQ, S2::G, S2::M>(nlist, elist, D, G, u, w, lam0, B, lam1, mask, st,
                                             partials, part_base, reduce_count, cstride, s);
    }
  }
  if constexpr (NQ >= 3 && NQ <= 15 && NQ != 4) {
    if (variant == 8 && ncomp == 1) {   // TMA-staged operands (bk5_stage.cuh)
      // cstride carries the length of the u array for ncomp = 1 (nk_bk5_batch)
      using SD = StageShapes<NQ>;
#define NK_SARGS nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials, part_base, \
                 reduce_count, cstride, s, nblocks
      if (cfg == 21) return runs<NQ, SD::G[1], SD::U[1], SD::M[1], SD::E[1]>(NK_SARGS);
      if (cfg == 22) return runs<NQ, SD::G[2], SD::U[2], SD::M[2], SD::E[2]>(NK_SARGS);
      return runs<NQ, SD::G[0], SD::U[0], SD::M[0], SD::E[0]>(NK_SARGS);
#undef NK_SARGS
    }
  }
  if (variant == 5 && ncomp == 1)
    return run_pencil2<NQ>(cfg, nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials,
                           part_base, reduce_count, s, nblocks, pf_dist);
  if ((variant == 3 || variant == 4) && ncomp == 1)
    return run_pencil<NQ>(cfg, nlist, elist, D, G, u, w, lam0, B, lam1, mask, st, partials,
                          part_base, reduce_count, s, nblocks, pf_dist);
  if (ncomp == 1)
    return run_cfg<NQ, 1>(cfg, nlist, elist, D, G, u, w, lam0, B, lam1, cstride, mask, st,
                          partials, part_base, reduce_count, s, nblocks, pf_dist);
  return run_cfg<NQ, 3>(cfg, nlist, elist, D, G, u, w, lam0, B, lam1, cstride, mask, st, partials,
                        part_base, reduce_count, s, nblocks, pf_dist);
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

// the stage kernel with the PCG head fused (bk5_stage.cuh, PCG = true) at
// N + 1 in 9..15: whole-array steps only (u_len = nlist elements)
constexpr int kNotServed = -1000;
template <int NQ>
static int run_stage_pcg(int64_t nlist, const double* D, const double* G, double* p, double* w,
                         double lam0, const double* B, double lam1, const uint8_t* mask,
                         double* x, const double* r, const double* invD, nk_cg_state* st,
                         double* partials, int64_t part_base, int64_t reduce_count,
                         double* hist, cudaStream_t s, int64_t* nblocks) {
  if constexpr (NQ >= 9 && NQ <= 15) {
    using SD = StageShapes<NQ>;
    static_assert(SD::U[0] == 2 && SD::E[0] == 1, "stage PCG: two u buffers, one element");
    if (nblocks) {
      *nblocks = stage_pcg_grid<NQ, SD::G[0], SD::M[0]>(nlist);
      return NK_OK;
    }
    return launch_stage_pcg<NQ, SD::G[0], SD::M[0]>(nlist, D, G, p, w, lam0, B, lam1, mask, x, r,
                                                    invD, st, partials, part_base, reduce_count,
                                                    hist, s);
  } else {
    return kNotServed;
  }
}

extern "C" int NK_CAT(nk_bk5_pcg_nq, NK_BK5_NQ)(int64_t nlist, const int32_t* elist,
                                               const double* D, const double* G, double* p,
                                               double* w, double lam0, const double* B,
                                               double lam1, const uint8_t* mask, double* x,
                                               const double* r, const double* invD,
                                               nk_cg_state* st, double* partials,
                                               int64_t part_base, int64_t reduce_count,
                                               double* hist, cudaStream_t s, int64_t* nblocks) {
  constexpr int NQ = NK_BK5_NQ;
  constexpr int EPB = PencilDefault<NQ>::EPB;
  constexpr int MINB = NQ == 8 ? 10 : PencilDefault<NQ>::MINB;  // ~100 regs at NQ = 8
  if constexpr (NQ == 2) {   // point per thread (the order-1 coarse level)
    const int64_t nb = (nlist * 8 + kN1PtThreads - 1) / kN1PtThreads;
    if (nblocks) {
      *nblocks = nb;
      return NK_OK;
    }
    if (nb == 0) return NK_OK;
    DParam<2> Dp;
    Dp.set(D);
    bk5_n1_pcg<2><<<(unsigned)nb, kN1PtThreads, 0, s>>>(nlist, elist, Dp, G, p, w, lam0, B, lam1,
                                                   mask, x, r, invD, st, partials, part_base,
                                                   reduce_count, hist);
    return check_launch("bk5_n1_pcg");
  }
  if constexpr (NQ == 8) {
    if (nk_bk5_variant_get() != 3) {  // auto / 4: TMA pipeline
      if (knob(NK_KNOB_TMA) == 2) {  // single p / G buffers, four CTAs per SM
        if (nblocks) {
          *nblocks = tma_pcg_grid<NQ, 4, true>(nlist);
          return NK_OK;
        }
        return launch_pencil_tma_pcg<NQ, 4, true>(nlist, elist, D, G, p, w, lam0, B, lam1, mask,
                                                  x, r, invD, st, partials, part_base,
                                                  reduce_count, hist, s);
      }
      if (knob(NK_KNOB_TMA) == 1) {  // single p / G buffers, five CTAs per SM
        if (nblocks) {
          *nblocks = tma_pcg_grid<NQ, 5, true>(nlist);
          return NK_OK;
        }
        return launch_pencil_tma_pcg<NQ, 5, true>(nlist, elist, D, G, p, w, lam0, B, lam1, mask,
                                                  x, r, invD, st, partials, part_base,
                                                  reduce_count, hist, s);
      }
      if (nblocks) {
        *nblocks = tma_pcg_grid<NQ, 3>(nlist);
        return NK_OK;
      }
      return launch_pencil_tma_pcg<NQ, 3>(nlist, elist, D, G, p, w, lam0, B, lam1, mask, x, r,
                                          invD, st, partials, part_base, reduce_count, hist, s);
    }
  }
  {
    const int v = nk_bk5_variant_get();
    if (elist == nullptr && knob(NK_KNOB_STAGE_PCG) && (v == 0 || v == 8)) {
      const int rc = run_stage_pcg<NQ>(nlist, D, G, p, w, lam0, B, lam1, mask, x, r, invD, st,
                                       partials, part_base, reduce_count, hist, s, nblocks);
      if (rc != kNotServed) return rc;
    }
  }
  if (nblocks) {
    *nblocks = (nlist + EPB - 1) / EPB;
    return NK_OK;
  }
  return launch_pencil_pcg<NQ, EPB, MINB>(nlist, elist, D, G, p, w, lam0, B, lam1, mask, x, r,
                                          invD, st, partials, part_base, reduce_count, hist, s);
}
