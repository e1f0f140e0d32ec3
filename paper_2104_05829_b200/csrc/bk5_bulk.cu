// BK5 variant 2: persistent CTAs with a cp.async.bulk (TMA 1-D) pipeline.
// (placeholder until implemented; variant 1 serves every order)
#include "common.cuh"

static int g_variant = 0;  // 0 auto (pencil), 1 k-slab, 2 bulk, 3 pencil

extern "C" int nk_bk5_variant_get() { return g_variant; }

extern "C" int nk_bk5_set_variant(int v) {
  int old = g_variant;
  g_variant = v;
  return old;
}

extern "C" int nk_bk5_bulk_launch(int N, int64_t nlist, const int32_t* elist, const double* D,
                                  const double* G, const double* u, double* w, double lam0,
                                  const double* B, double lam1, const uint8_t* mask,
                                  nk_cg_state* st, double* partials, int64_t part_base,
                                  int64_t reduce_count, cudaStream_t s, int64_t* nblocks_out,
                                  int query_only) {
  nk::set_error("bk5 bulk variant not built");
  return NK_ERR_UNSUPPORTED;
}
