// Process-wide BK5 variant selection (nk_bk5_set_variant, include/nekb200.h):
// 0 auto (the measured per-order table in bk5.cu), 1 k-slab, 3 pencil,
// 4 pencil-TMA, 5 pencil2, 6 seq3 (3-component batches; scalar calls use
// the auto table).
#include "common.cuh"

static int g_variant = 0;

extern "C" int nk_bk5_variant_get() { return g_variant; }

extern "C" int nk_bk5_set_variant(int v) {
  int old = g_variant;
  g_variant = v;
  return old;
}
