// Process-wide BK5 variant selection (nk_bk5_set_variant, include/nekb200.h):
// 0 auto (the measured per-order table in bk5.cu), 1 k-slab, 3 pencil,
// 4 pencil-TMA, 5 pencil2, 6 seq3 (3-component batches; scalar calls use
// the auto table), 7 dmma, 8 stage (TMA-staged operands, N + 1 in 8..15).
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
// follow, 0.117 -> 0.127 ms), and a one-trip-ahead L2 prefetch in the update;
// L2 hints: streamed data evict_first + r / w evict_last (0.1136 -> 0.1101 ms,
// profiles/r2l_bp5_knobs.jsonl; the persisting set-aside did not help, r2m);
// the N = 7 TMA step with single p / G buffers at four CTAs per SM (0.1080 ->
// 0.1068 ms, profiles/r2zo_bp5_tma_knob.jsonl); the fused gs update
// software-pipelined two deep (0.1066 -> 0.1049 ms, r2zp_bp5_cg_pipe.jsonl)
// on a 4 x 148-block grid for every CG vector kernel (N = 3: 0.0330 ->
// 0.0309 ms, N = 9: 0.2235 -> 0.2171 ms, N = 7 neutral; r2zr_bp5_vec_grid.jsonl).
static int g_knobs[NK_KNOB_COUNT] = {nk::kPdlStep | nk::kPdlVec, 1,
                                     nk::kL2StreamFirst | nk::kL2ReuseLast, 2, 2, 6, 1, 0};

namespace nk {
int knob(int k) { return (k >= 0 && k < NK_KNOB_COUNT) ? g_knobs[k] : 0; }

static const GsTail* g_tail = nullptr;
static bool g_tail_used = false;
const GsTail* gs_tail_offer() { return g_tail; }
void gs_tail_set(const GsTail* t) {
  g_tail = t;
  g_tail_used = false;
}
void gs_tail_mark_used() { g_tail_used = true; }
bool gs_tail_used() { return g_tail_used; }

static const unsigned long long* g_gate = nullptr;
const unsigned long long* bk5_gate() { return g_gate; }
void set_gate_ptr(const void* p) { g_gate = static_cast<const unsigned long long*>(p); }

void l2_apply_set_aside() {
  static int applied = 0;   // the device default: no set-aside
  const int want = (g_knobs[NK_KNOB_L2] & kL2SetAside) ? 1 : 0;
  if (want == applied) return;
  int dev = 0, maxp = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want ? (size_t)maxp : 0);
  cudaGetLastError();
  applied = want;
}
}  // namespace nk

extern "C" int64_t nk_l2_set_aside_max() {
  int dev = 0, maxp = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess)
    return -1;
  return maxp;
}

extern "C" int nk_set_knob(int k, int value) {
  if (k < 0 || k >= NK_KNOB_COUNT) {
    nk::set_error("set_knob: unknown knob %d", k);
    return -1;
  }
  const int old = g_knobs[k];
  g_knobs[k] = value;
  if (k == NK_KNOB_L2) nk::l2_apply_set_aside();   // a host call: never inside a capture
  return old;
}

extern "C" int nk_bk5_set_gate(const void* gate) {
  nk::set_gate_ptr(gate);
  return NK_OK;
}
