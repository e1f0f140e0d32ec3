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

// Knobs (NK_KNOB_*): defaults are the measured best (profiles/r2j_bp5_knobs.jsonl:
// BP5 N = 7, E = 20^3: 0.1175 -> 0.1152 ms per iteration; N = 3: 0.0378 ->
// 0.0360): PDL for the BK5 step and the CG vector kernels, not for the gs
// classes kernel (whose early-resident CTAs slow the step kernel they
// follow, 0.117 -> 0.127 ms), and a one-trip-ahead L2 prefetch in the update.
static int g_knobs[NK_KNOB_COUNT] = {nk::kPdlStep | nk::kPdlVec, 1};

namespace nk {
int knob(int k) { return (k >= 0 && k < NK_KNOB_COUNT) ? g_knobs[k] : 0; }
}  // namespace nk

extern "C" int nk_set_knob(int k, int value) {
  if (k < 0 || k >= NK_KNOB_COUNT) {
    nk::set_error("set_knob: unknown knob %d", k);
    return -1;
  }
  const int old = g_knobs[k];
  g_knobs[k] = value;
  return old;
}
