/*
 * nekb200.h -- C ABI of libnekb200.so, the B200 (sm_100a) hot path of the
 * spectral-element Poisson/Helmholtz operator  w_L = QQ^T Z_L u_L  inside PCG
 * (arXiv 2104.05829, NekRS).
 *
 * The reference (/root/reference) is a Python package, `nekmini`, whose
 * operator API is specified in SPEC.md; it has no FFI of its own.  Each entry
 * point below replaces one SPEC operation (cited per function).  The Python
 * mirror of the SPEC API (paper_2104_05829_b200/) binds these with ctypes;
 * INTEGRATION.md shows the binding a nekmini maintainer would add.
 *
 * Conventions (all functions):
 *   - return NK_OK (0) on success, a positive NK_ERR_* code otherwise; the
 *     message is available from nk_last_error() (thread-local).  Nothing
 *     throws across the ABI.
 *   - every pointer argument marked [dev] is a device pointer owned by the
 *     caller (torch allocates; the library never allocates or frees caller
 *     buffers).  [host] pointers are host memory.
 *   - every kernel is enqueued on `stream` (a cudaStream_t); nothing
 *     synchronises the host.  Scalars that drive the solver (alpha, beta,
 *     convergence) live in device memory (nk_cg_state), so whole PCG
 *     iterations can be captured in a CUDA graph.
 *   - Field layout: element-major FP64,
 *     u[e][k][j][i] with i fastest; vector fields component-major.
 *     Geometric factors G[e][6][(N+1)^3] in the order G11 G12 G13 G22 G23 G33
 *     (SPEC.md:102); mass B[e][(N+1)^3].
 *   - local point indices are int32: at most 2^31-1 local points per rank.
 */
#ifndef NEKB200_H
#define NEKB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* nk_stream_t; /* cudaStream_t */

enum {
  NK_OK = 0,
  NK_ERR_INVALID = 1,     /* contract error: bad size / order / pointer     */
  NK_ERR_CUDA = 2,        /* CUDA runtime error (launch, no device, ...)     */
  NK_ERR_UNSUPPORTED = 3, /* order N outside the compiled range             */
};

/* reduction ops of gs_op */
enum { NK_OP_ADD = 0, NK_OP_MUL = 1, NK_OP_MIN = 2, NK_OP_MAX = 3 };

/* deformation kinds of build_box_mesh */
enum { NK_DEFORM_NONE = 0, NK_DEFORM_SINE = 1 };

/* Device-resident PCG scalars.  Allocate sizeof(nk_cg_state) bytes of device
 * memory ZERO-INITIALISED once (the Python side uses a uint8 tensor; the
 * last-block tickets must start at 0 and reset themselves), then start each
 * solve with nk_cg_init / nk_cg_init_finalize. */
typedef struct {
  double rz;       /* <r, z>_w of the current iterate                        */
  double pAp;      /* <p, A p>  (rank-local sum until all-reduced)           */
  double rz_new;   /* <r_new, z_new>_w                                       */
  double rr;       /* <r_new, r_new>_w  (assembled residual norm^2)          */
  double zap;      /* <z_new, A p>_w  (flexible PCG only)                    */
  double bb;       /* <b, b>_w                                               */
  double thresh2;  /* tol^2 * bb                                             */
  double alpha;    /* last alpha (diagnostic)                                */
  int32_t iter;    /* completed iterations                                   */
  int32_t done;    /* 1 once converged, broken down or out of iterations     */
  int32_t converged;
  int32_t breakdown;
  int32_t max_iter;
  int32_t flexible;
  uint32_t ticket[4]; /* last-block-done counters (self-resetting)           */
  uint32_t gen;       /* grid-barrier generation (nk_bk5_pcg_gs; monotonic)   */
  uint32_t pad_;
} nk_cg_state;

/* ------------------------------------------------------------------ misc */
int nk_version(void);
const char* nk_last_error(void);
/* compiled orders: N in [NK_MIN_ORDER, NK_MAX_ORDER] */
int nk_order_range(int* nmin, int* nmax);
/* SM count and L2 size of the current device */
int nk_device_info(int* sm_count, int64_t* l2_bytes, int* cc_major, int* cc_minor);
/* L2 flush between timed reps: write the first half of `buf` [dev], then
 * read the second half, so L2 ends cold AND clean (each half should exceed
 * the 126 MB L2). */
int nk_l2_flush(void* buf, int64_t bytes, nk_stream_t stream);

/* diagnostic: BK5's HBM byte pattern without the arithmetic (read u and the
 * six G factors of every element, write w); nq3 even. */
int nk_bw_probe(int64_t nelem, int nq3, const double* u, const double* G, double* w,
                int blocks_per_sm, nk_stream_t stream);

/* ------------------------------------------------------------- geometry
 * build_box_mesh / geometric_factors on device.          */

/* GLL point coordinates xyz[3][nelem][(N+1)^3] [dev] of box elements.
 * elem_index [dev, nullable]: global element index of each local element
 * (e = ex + nx*(ey + ny*ez)); NULL means 0..nelem-1.  counts/extent/origin
 * [host, 3 each]; nodes [dev] = GLL nodes of order N (upload the basis
 * array; nothing is re-derived on device).  Replaces the coordinate part of
 * build_box_mesh. */
int nk_box_coords(int N, int64_t nelem, const int64_t* elem_index, const int32_t* counts,
                  const double* extent, const double* origin, int deform_kind, double amp,
                  const double* nodes, double* xyz, nk_stream_t stream);

/* G[nelem][6][(N+1)^3], B[nelem][(N+1)^3], optional J and metrics
 * rx[3][3][nelem][(N+1)^3] (rx[q][c] = dr_q/dx_c) [dev] from coordinates via
 * dx/dr = D_q x (geometric_factors).
 * status [dev, 2 x int64, caller-initialised to INT64_MAX]: status[0] = lowest
 * element with |J| < 1e-14 (degenerate), status[1] = lowest with J <= 0
 * (inverted). */
int nk_geom_factors(int N, int64_t nelem, const double* D, const double* weights,
                    const double* xyz, double* G, double* B, double* J, double* rx,
                    int64_t* status, nk_stream_t stream);

/* Global ids of box points (assign_global_ids for generated boxes,
 * SPEC.md:138-146): rank of the undeformed lattice point in (z,y,x) order,
 * 1-based.  periodic [host, 3 x int32]. */
int nk_box_ids(int N, int64_t nelem, const int64_t* elem_index, const int32_t* counts,
               const int32_t* periodic, int64_t* ids, nk_stream_t stream);

/* Dirichlet mask: mask[e][k][j][i] = 0 on faces whose
 * dirichlet[f] != 0 (faces x-,x+,y-,y+,z-,z+; [host, 6 x int32]), else 1. */
int nk_box_mask(int N, int64_t nelem, const int64_t* elem_index, const int32_t* counts,
                const int32_t* dirichlet, uint8_t* mask, nk_stream_t stream);

/* ------------------------------------------------------------------ BK5
 * apply_stiffness_local + Helmholtz/mass term
 * (SPEC.md:380-388, 403):
 *     w_e = lam0 * sum_{mm'} D_m^T G_mm' D_m' u_e  +  lam1 * B_e u_e
 * for the elements in elem_list [dev, int32, nullable = all nelem], with
 * D [HOST] the (N+1)x(N+1) D-hat (row-major D[a][i] = h_i'(xi_a)); it is
 * copied by value into the launch parameters (so a captured CUDA graph keeps
 * it) and read by the kernels from the constant bank.
 * ncomp components are batched (G read once): u, w, B-scaled fields at
 * comp_stride doubles apart.  mask [dev u8, nullable]: w *= mask.
 * Fused PCG dot (pass st != NULL): if st->done the launch is a no-op;
 * otherwise each block writes sum(u * w) to partials[part_base + block] and,
 * when reduce_count > 0, the last block sums partials[0 .. reduce_count) in
 * fixed order into st->pAp (= p^T A p, since sum_L p_L (A_L p)_L =
 * p^T Q^T A_L Q p for continuous p).  nk_bk5_blocks() tells how many blocks a
 * launch uses. */
int nk_bk5(int N, int64_t nelem, const double* D, const double* G, const double* u,
           double* w, double lam0, const double* B, double lam1, int ncomp,
           int64_t comp_stride, const uint8_t* mask, const int32_t* elem_list, int64_t nlist,
           nk_cg_state* st, double* partials, int64_t part_base, int64_t reduce_count,
           nk_stream_t stream);
int64_t nk_bk5_blocks(int N, int64_t nlist, int ncomp);
/* nk_bk5 for a 3-component batch with per-component fused dots (the batched
 * vector-Helmholtz PCG, configs[4]; "geometric factors ...
 * reused across each velocity component"): st points to ncomp CG states;
 * component c's block partials of p_c . A p_c go to partials + c *
 * part_stride (part_stride >= reduce_count) and its sum to st[c].pAp; a
 * component whose state is done is skipped.  Runs seq3 (G from HBM once for
 * the three components) where nk_bk5_batch_variant(N) == 6, else three
 * scalar launches.  With st == NULL it is nk_bk5. */
int nk_bk5_batch(int N, int64_t nelem, const double* D, const double* G, const double* u,
                 double* w, double lam0, const double* B, double lam1, int ncomp,
                 int64_t comp_stride, const uint8_t* mask, const int32_t* elem_list,
                 int64_t nlist, nk_cg_state* st, double* partials, int64_t part_stride,
                 int64_t part_base, int64_t reduce_count, nk_stream_t stream);
/* the 3-component kernel nk_bk5 / nk_bk5_batch run at order N: 6 = seq3,
 * 3 = pencil3, -1 = three scalar launches (the measured auto table). */
int nk_bk5_batch_variant(int N);
/* blocks of one nk_bk5_batch launch (ncomp = 3, with st) over nlist elements
 * -- the reduce_count of a single launch, the minimum part_stride. */
int64_t nk_bk5_batch_blocks(int N, int64_t nlist);
/* kernel variant selection: 0 = auto (measured per-order table: 8 for
 * N in {6,8,9,10,12,13,14,15}, 5 for N = 2, else 3; 3-component batches:
 * 6 at N in {3,5,7..13}, pencil3 at N in {4,6}, three scalar launches
 * elsewhere), 5 = pencil2 (two shared buffers, u re-read from L1/L2), 1 =
 * k-slab (2D thread plane, k-column in registers, D in shared memory), 3 =
 * pencil (register 1-D contractions, D in the constant bank, swizzled shared
 * transposes), 4 = pencil-TMA (persistent CTAs, cp.async.bulk 2-stage ring;
 * N+1 in {4, 6, 8}, else pencil), 6 = seq3 (ncomp = 3: the pencil kernel
 * running the three components back to back per CTA, G from HBM once;
 * ncomp = 1 calls use the auto table), 7 = dmma (FP64 tensor-core
 * contractions, N+1 in 9..16), 8 = stage (persistent CTAs; the next
 * element's u and G moved into shared memory by cp.async.bulk while the
 * current one computes, w assembled in shared memory and bulk-stored,
 * several elements per CTA below N = 7; N+1 in 3, 5..16, else pencil),
 * 9 = stage2 (stage with two threads per pencil, N+1 in 9..15), 10 = pair
 * (one element per thread-block cluster of two CTAs split by k-planes:
 * multicast u, all six G components staged, gt exchanged through
 * distributed shared memory; N+1 = 16), 11 = point (one thread per point,
 * element groups staged by cp.async.bulk; N+1 = 3, whole-array calls with
 * 16-byte aligned u and G, else pencil2).  N = 1 always runs its point-per-lane kernel
 * unless 1 is set.  Variants 3/4/5/7/8 serve ncomp = 1; with them forced,
 * ncomp = 3 uses pencil3 (k-slab for 1) or three scalar launches.  Returns
 * the previous value. */
int nk_bk5_set_variant(int variant);
/* shape tuning: cfg selects the (elements per CTA, CTAs per SM) shape --
 * k-slab at N = 7 (0 = default 4x2, 1 = 4x3, 2 = 2x4, 3 = 2x6, 4 = 1x8,
 * 5 = 1x12, 6 = 8x1), pencil at N = 7 (1..9, bk5_inst.cu), and pencil /
 * pencil2 at N = 2..6, 8..15 (11..14: the PencilAlt table in bk5_inst.cu,
 * swept by scripts/bk5_sweep.py --high-shapes); pf_dist = L2 bulk-prefetch distance in CTAs (-1 = one wave of
 * resident CTAs ahead, 0 = off). */
int nk_bk5_tune(int cfg, int pf_dist);

/* process-wide knobs; returns the previous value, or -1 for an unknown knob.
 *   NK_KNOB_PDL: 1 = launch the PCG-iteration kernels (fused / split BK5
 *     step, gs classes, CG updates) with programmatic dependent launch: each
 *     kernel is scheduled while its predecessor drains, runs its static-
 *     operand prologue (G bulk copies, plan indices, gs codes), then waits
 *     for the predecessor's results (griddepcontrol.wait); 0 = plain launches.
 *   NK_KNOB_CG_UPDATE: nk_cg_update_gs 16-B kernel -- k > 0 = each block
 *     bulk-prefetches (cp.async.bulk.prefetch.L2) its r / w / invD / code
 *     segment k grid-stride trips ahead; 0 = no prefetch.  Bit-identical.
 *   NK_KNOB_L2: L2 eviction-priority hints in the BP5 step and update
 *     kernels -- bit 1: data streamed once per iteration (G, p, x, codes,
 *     mask) evict_first; bit 2: r and w (reused by the next kernel) evict_last;
 *     bit 4: invD (read twice per iteration) evict_last; bit 8: reserve the
 *     device's maximum persisting-L2 set-aside for the evict_last lines
 *     (cudaLimitPersistingL2CacheSize; released when the bit is cleared).
 *     Bit-identical.
 *   NK_KNOB_FDM: nk_fdm (FP64) contractions -- 1 = FP64 tensor cores
 *     (mma.sync m8n8k4, N + 3 <= 16), 0 = the CUDA-core line kernel, 2 =
 *     (default) the measured winner per order (tensor cores at N = 4, 5,
 *     9..13).  Same algorithm, sums in a different order (rounding-level
 *     differences).
 *   NK_KNOB_TMA: the order-7 TMA BP5 step kernel -- 0 = two-stage (p, G)
 *     ring, three CTAs per SM; 1 = single p and G buffers refilled as soon
 *     as each is consumed, five CTAs per SM (200 registers); 2 = (default)
 *     single buffers, four CTAs per SM.  Same arithmetic per element; the
 *     grid (and so the grouping of the p.Ap partial sums) follows the CTAs
 *     per SM.
 *   NK_KNOB_CG_PIPE: bits 0-1: nk_cg_update_gs 16-B kernel -- 1 =
 *     software-pipelined across grid-stride trips (the next trip's code /
 *     invD / r / w loaded while the current trip's partner gather runs); 2 =
 *     two deep (codes two trips ahead, partner values one trip ahead); 0 =
 *     per-trip loads (bit-identical to each other).  Bit 4: the CG vector
 *     kernels' grid capped at 4 x 148 blocks instead of 8 x 148 (a different
 *     but still fixed, device-independent grouping of the dot partial sums).
 *     Default 6.  Applies to vectors of up to 2^24 points; larger ones (HBM-
 *     streamed, not L2-resident) always run the per-trip form on 8 x 148
 *     blocks (measured faster there).
 *   NK_KNOB_STAGE_PCG: nk_bk5_pcg at N + 1 in 9..15 (no element list) -- 1 =
 *     the stage kernel with the Jacobi-PCG head fused into its F3 pass
 *     (TMA-staged p and G); 0 = the register-pencil fused step.
 *   NK_KNOB_GS_TAIL: nk_bk5_pcg_gs -- 1 = fold the edge / vertex gs into
 *     the persistent N = 7 TMA step behind a grid barrier (one launch,
 *     bit-identical); 0 (default: measured 5-7% slower per BP5 iteration
 *     in graph replay, profiles/r2zzc_gs_tail_ab.jsonl) = nk_bk5_pcg
 *     followed by nk_gs_op_classes.  2 = nk_cg_update_gs_cls runs the same
 *     gs at the start of the update kernel (grid barrier, then the update). */
enum { NK_KNOB_PDL = 0, NK_KNOB_CG_UPDATE = 1, NK_KNOB_L2 = 2, NK_KNOB_FDM = 3,
       NK_KNOB_TMA = 4, NK_KNOB_CG_PIPE = 5, NK_KNOB_STAGE_PCG = 6, NK_KNOB_GS_TAIL = 7,
       NK_KNOB_COUNT = 8 };
int nk_set_knob(int knob, int value);
/* chunk-gated stage BK5 (the host-buffer e2e stream, kernels.py
 * _HostStream): while set (non-null), stage-kernel launches (variant 8, no
 * element list) wait before staging element e's u until the device u64 at
 * `gate` is >= e + 1 -- the copy engine writes there the element count each
 * H2D chunk completes, so one persistent kernel consumes the chunks as they
 * land.  The pointer is captured into the launch (CUDA graphs keep it);
 * set nullptr afterwards.  A gate that never arrives times out after ~2 s
 * (wrong results, no hang). */
int nk_bk5_set_gate(const void* gate);
/* stream-ordered 64-bit write of `value` to device memory `dptr` by the GPU
 * front end (cuStreamWriteValue64), after all prior work on `stream`; the
 * chunk gate's writer (no copy engine, no SM; graph-capturable). */
int nk_stream_write_u64(void* dptr, uint64_t value, nk_stream_t stream);
/* the device's maximum persisting-L2 set-aside in bytes (-1: no device). */
int64_t nk_l2_set_aside_max(void);

/* Fused BP5 operator step (pcg iteration k = st->iter):
 *   k > 0: stop if st->rr <= st->thresh2 or k >= max_iter (sets done,
 *          converged, hist[k]); x += alpha_{k-1} p (deferred x update);
 *          p = invD r + beta p  (Fletcher-Reeves, or flexible beta)
 *   w = mask * (lam0 A_L p + lam1 B p); st->pAp = sum_L p w  (last block)
 * p, x updated in place [dev].  Follow with gs(w) and nk_cg_update with
 * x = NULL, p = NULL (which advances st->iter).  partials:
 * nk_bk5_pcg_blocks(N, nlist) doubles per launch (offset part_base). */
int nk_bk5_pcg(int N, int64_t nelem, const double* D, const double* G, double* p, double* w,
               double lam0, const double* B, double lam1, const uint8_t* mask,
               const int32_t* elem_list, int64_t nlist, double* x, const double* r,
               const double* invD, nk_cg_state* st, double* partials, int64_t part_base,
               int64_t reduce_count, double* hist, nk_stream_t stream);
int64_t nk_bk5_pcg_blocks(int N, int64_t nlist);
/* nk_bk5_pcg over all elements (no element list) followed by the
 * gather-scatter (+) of w over a classes plan -- on one rank, the >= 3-member
 * (edge / vertex) segments that nk_cg_update_gs leaves out (SPEC.md:479-487:
 * the operator + gs_op pair of one PCG iteration; the class table is
 * nk_gs_op_classes's).  Where the step kernel is persistent (N = 7 TMA step,
 * NK_KNOB_GS_TAIL) the gs runs inside it after a grid barrier, in the same
 * lane order and fold as nk_gs_op_classes -- bit-identical, one launch
 * fewer; otherwise the two launches.  Returns nk_bk5_pcg's status. */
int nk_bk5_pcg_gs(int N, int64_t nelem, const double* D, const double* G, double* p, double* w,
                  double lam0, const double* B, double lam1, const uint8_t* mask, double* x,
                  const double* r, const double* invD, nk_cg_state* st, double* partials,
                  int64_t reduce_count, double* hist, int nclass, const int32_t* sizes,
                  const int64_t* nsegs, const int32_t* const* members, nk_stream_t stream);
/* 1 if nk_bk5_pcg_gs at order N runs as one launch under the current knobs */
int nk_bk5_pcg_gs_fused(int N);

/* closed-form diag(lam0*A_e + lam1*B_e) per element (extract_diagonal
 * before assembly) */
int nk_local_diag(int N, int64_t nelem, const double* D, const double* G, double lam0,
                  const double* B, double lam1, double* diag, nk_stream_t stream);

/* ------------------------------------------------------ gather-scatter
 * gs_op(handle, w, op) on one rank: for each segment s,
 * the values w[perm[seg_start[s]] .. perm[seg_start[s+1]-1]] are folded
 * sequentially in that (canonical: ascending local index) order and the
 * result written back to every member.  Points outside all segments are
 * untouched.  ncomp fields at comp_stride apart share one plan.
 * st [nullable]: skip when st->done (PCG graph replays). */
int nk_gs_op(int64_t nseg, const int32_t* seg_start, const int32_t* perm, double* w, int op,
             int ncomp, int64_t comp_stride, const nk_cg_state* st, nk_stream_t stream);

/* The same plan re-packed by multiplicity class (one launch for all
 * classes, at most 16, segment size 1..32): class c has segment size
 * sizes[c] [host] and nsegs[c] [host] segments whose members are members[c]
 * [host array of dev pointers]: int32, segment-major, each segment padded to
 * Mp = next power of two >= sizes[c] with -1 (members[c][s * Mp + m]),
 * members in canonical (ascending local index) order.  One lane per member;
 * fold via warp shuffles in member order: bit-identical to nk_gs_op. */
int nk_gs_op_classes(int nclass, const int32_t* sizes, const int64_t* nsegs,
                     const int32_t* const* members, double* w, int op, int ncomp,
                     int64_t comp_stride, const nk_cg_state* st, nk_stream_t stream);

/* 32-bit gs_op (SPEC.md:202's precision = 32-bit): the same plans and the
 * same canonical fold order on float fields (folded in FP32). */
int nk_gs_op_f32(int64_t nseg, const int32_t* seg_start, const int32_t* perm, float* w, int op,
                 int ncomp, int64_t comp_stride, const nk_cg_state* st, nk_stream_t stream);
int nk_gs_op_classes_f32(int nclass, const int32_t* sizes, const int64_t* nsegs,
                         const int32_t* const* members, float* w, int op, int ncomp,
                         int64_t comp_stride, const nk_cg_state* st, nk_stream_t stream);

/* Host-side plan construction (gs_setup for one rank):
 * stable counting sort of ids [host, n] by id; ids with multiplicity >= 2
 * become segments.  perm [host, capacity n], seg_start [host, capacity
 * n/2 + 2].  Ids <= 0 are singletons.  Writes counts to *nseg, *nperm. */
int nk_gs_plan_build(const int64_t* ids, int64_t n, int32_t* perm, int32_t* seg_start,
                     int64_t* nseg, int64_t* nperm);

/* Library-owned gs handle (SPEC.md:184-200 GatherScatterHandle, one rank):
 * built from the canonical CSR of nk_gs_plan_build [host perm, seg_start],
 * re-packed by multiplicity class on the device.  nk_gs_apply runs the
 * same bit-exact canonical fold as nk_gs_op / nk_gs_op_classes (the SURVEY
 * sketch's nk_gs_op(handle, ...)); handles are not thread-safe and must be
 * destroyed with nk_gs_destroy. */
typedef struct nk_gs nk_gs;
int nk_gs_create(const int32_t* perm, const int32_t* seg_start, int64_t nseg, int64_t nperm,
                 nk_gs** out);
int nk_gs_apply(nk_gs* h, double* w, int op, int ncomp, int64_t comp_stride,
                const nk_cg_state* st, nk_stream_t stream);
int nk_gs_destroy(nk_gs* h);

/* dst[i] = src[idx[i]] for i < n  (halo pack) */
int nk_gather(int64_t n, const int32_t* idx, const double* src, double* dst,
              const nk_cg_state* st, nk_stream_t stream);
/* Cross-rank combine (halo unpack): for each shared id h < nh,
 *   t = fold(buf[src_idx[src_start[h]]], ..., buf[src_idx[src_start[h+1]-1]])
 * in that order (ascending rank), then w[dst_idx[d]] = t for d in
 * [dst_start[h], dst_start[h+1]). */
int nk_halo_combine(int64_t nh, const int32_t* src_start, const int32_t* src_idx,
                    const double* buf, const int32_t* dst_start, const int32_t* dst_idx,
                    double* w, int op, const nk_cg_state* st, nk_stream_t stream);

/* ------------------------------------------- NVLink peer-memory halo
 * NCCL-free halo transport (gs_op_overlapped's exchange, SPEC.md:212-220;
 * PAPER.md:130-141): library-owned receive buffers mapped into the
 * neighbours through CUDA IPC; the push kernel stores boundary contributions
 * straight into the neighbour's buffer over NVLink and publishes a per-pair
 * epoch flag (system-scope release); the combine kernel acquire-waits on the
 * flags, then folds in canonical order.  Buffers are double-buffered by epoch
 * parity; epochs live in device memory (graph-replayable). */
int nk_ipc_handle_size(void);
/* cudaMalloc'ed, zeroed, IPC-exportable buffer; handle: nk_ipc_handle_size() bytes */
int nk_ipc_alloc(int64_t bytes, void** ptr, void* handle);
int nk_ipc_free(void* ptr);
int nk_ipc_open(const void* handle, void** peer_ptr);
int nk_ipc_close(void* peer_ptr);
/* for neighbour q < nnb (<= 8): peer_recv[q][par*recv_len[q] + recv_off[q] + i]
 * = w[send_idx[send_start[q] + i]]; par = (epoch[0]+1) & 1; then epoch[0]++
 * and *peer_flag[q] = epoch[0] (release.sys).  epoch [dev, 2 x u64, zeroed]. */
int nk_halo_push(int nnb, void* const* peer_recv, const int64_t* recv_off,
                 const int64_t* recv_len, void* const* peer_flag, const int32_t* send_start,
                 const int32_t* send_idx, const double* w, int64_t total, uint64_t* epoch,
                 const nk_cg_state* st, nk_stream_t stream);
/* wait flags[0..nflags) >= epoch[0] (acquire.sys), then as nk_halo_combine
 * with buf index s < own_len read from buf[s] and s >= own_len from
 * buf[par*buf_len + s]. */
int nk_halo_combine_wait(int64_t nh, const int32_t* src_start, const int32_t* src_idx,
                         const double* buf, int64_t buf_len, int64_t own_len,
                         const int32_t* dst_start, const int32_t* dst_idx, double* w, int op,
                         const uint64_t* flags, int nflags, const uint64_t* epoch,
                         const nk_cg_state* st, nk_stream_t stream);

/* Deterministic scalar all-reduce over peer memory (the PCG dots): vals[0..k)
 * [dev, k <= 4] are written into slot [parity][rank] of every rank's board
 * (boards[q] [host array of nranks mapped pointers, own included]) with a
 * release of flags_for_me[q]; then this rank acquire-waits on my_flags
 * [dev, nranks] and overwrites vals with the rank-ordered sum from my_board
 * [dev, 2 x nranks x 4 doubles].  Identical bits on every rank. */
int nk_board_allreduce(int nranks, int rank, double* vals, int k, void* const* boards,
                       void* const* flags_for_me, const double* my_board,
                       const uint64_t* my_flags, uint64_t* epoch, nk_stream_t stream);

/* --------------------------------------------------------------- PCG
 * Jacobi-PCG vector kernels (pcg).  Weighted dots use
 * wt [dev] = 1/multiplicity (so <a,b>_w is the assembled l2 product).
 * Every reduction is two-stage with a fixed order: run-to-run bitwise
 * deterministic.  partials [dev]: nk_cg_partials_len(n) doubles. */
int64_t nk_cg_partials_len(int64_t n);

/* x = 0, r = b, p = z = invD r; local sums bb, rr, rz into st.  Then (after
 * an optional all-reduce of st->{rz,rr,bb}) nk_cg_init_finalize sets
 * thresh2 = tol^2 bb and done/converged for b = 0 or r already small. */
int nk_cg_init(int64_t n, const double* b, double* x, double* r, double* p,
               const double* invD, const double* wt, nk_cg_state* st, double* partials,
               double tol, int max_iter, int flexible, nk_stream_t stream);
int nk_cg_init_finalize(nk_cg_state* st, double* hist, nk_stream_t stream);

/* alpha = rz/pAp (breakdown if pAp <= 0); x += alpha p; r -= alpha Ap;
 * local sums rr, rz_new (z = invD r; skipped if invD NULL), zap into st.
 * x = p = NULL selects the fused-BP5 form (x update deferred to nk_bk5_pcg;
 * advances st->iter).  Dot weights: wt [dev, FP64] if given, else
 * 1/mult with mult [dev, u8 multiplicity], else 1. */
int nk_cg_update(int64_t n, double* x, double* r, const double* p, const double* Ap,
                 const double* invD, const double* wt, const uint8_t* mult, nk_cg_state* st,
                 double* partials, nk_stream_t stream);

/* Single-rank fused-BP5 update with the face part of the gather-scatter
 * folded in: w is A p written by nk_bk5_pcg after a gs over the NON-PAIR
 * segments only (edges, vertices: nk_gs_op_classes on that sub-plan); each
 * point's assembled value and 1/mult dot weight come from its gs code
 * [dev, int32, n]: -1 unshared (w, 1); >= 0 the partner of a 2-member
 * segment (w + w[code], 1/2); <= -2 already assembled (w, 1/M with
 * M = -code).  Same sums as gs + nk_cg_update's fused form, bit for bit;
 * face pairs (most shared points) cost one L2 read instead of a gs pass.
 * Replaces the gs_op + cg_update pair of one PCG iteration
 * (SPEC.md:479-487). */
int nk_cg_update_gs(int64_t n, double* r, const double* w, const double* invD,
                    const int32_t* code, nk_cg_state* st, double* partials, nk_stream_t stream);

/* nk_gs_op_classes (+) on w over a classes plan -- the >= 3-member
 * segments -- followed by nk_cg_update_gs: under NK_KNOB_GS_TAIL = 2 (16-B
 * aligned r / w / invD, the pipelined update) ONE launch, the gs run by the
 * update kernel's grid before a grid barrier, bit-identical; otherwise the
 * two launches. */
int nk_cg_update_gs_cls(int64_t n, double* r, double* w, const double* invD, const int32_t* code,
                        int nclass, const int32_t* sizes, const int64_t* nsegs,
                        const int32_t* const* members, nk_cg_state* st, double* partials,
                        nk_stream_t stream);
/* 1 if nk_cg_update_gs_cls on n points is one launch under the current
 * knobs (16-byte aligned operands assumed) */
int nk_cg_update_gs_cls_fused(int64_t n);

/* The vector head of nk_bk5_pcg as its own coalesced pass (iteration
 * k = st->iter): k > 0: stop test on st->rr, x += alpha_{k-1} p,
 * p = invD r + beta p (Fletcher-Reeves or flexible beta); hist[k], stop and
 * rz bookkeeping as nk_bk5_pcg.  Follow with nk_bk5(..., st, partials) for
 * w = mask A p and st->pAp, then gs + nk_cg_update_gs as in the fused
 * schedule.  Used by FusedPCG at orders where it beats the
 * fused kernel (paper_2104_05829_b200/solvers.py). */
/* Batched forms (the lockstep 3-component PCG): ncomp components at
 * cstride in r / w (and x / p), states st[0..ncomp), partials at c * 3 *
 * nk_cg_partials_len(n) / 3 (i.e. 3 x 1184 doubles per component), history
 * hist + c * hstride; invD and code shared.  Each component advances, stops
 * and counts its own iterations. */
int nk_cg_update_gs_batch(int64_t n, int ncomp, int64_t cstride, double* r, const double* w,
                          const double* invD, const int32_t* code, nk_cg_state* st,
                          double* partials, nk_stream_t stream);
/* nk_cg_update_gs_batch with gathered segments: a code <= -NK_GS_SEG_BASE
 * marks a point of a rank-private segment of M >= 3 members listed at
 * segtab[k] = M, segtab[k+1..k+M] = its members in canonical (ascending
 * local index) order, k = -code - NK_GS_SEG_BASE; the point's assembled
 * value is the canonical fold of the members' w, computed in place -- so no
 * gs pass over edges / vertices precedes the update (bit-identical to one).
 * Codes -2 .. -(NK_GS_SEG_BASE-1) keep their meaning (-M: assembled before
 * the update, e.g. halo ids).  segtab NULL = nk_cg_update_gs_batch.  Needs
 * 16-byte aligned r / w / invD and 8-byte aligned code when segtab != NULL. */
#define NK_GS_SEG_BASE 65536
int nk_cg_update_gs_seg(int64_t n, int ncomp, int64_t cstride, double* r, const double* w,
                        const double* invD, const int32_t* code, const int32_t* segtab,
                        nk_cg_state* st, double* partials, nk_stream_t stream);
int nk_cg_xpstep_batch(int64_t n, int ncomp, int64_t cstride, double* x, const double* r,
                       double* p, const double* invD, nk_cg_state* st, double* hist,
                       int64_t hstride, nk_stream_t stream);
int nk_cg_xpstep(int64_t n, double* x, const double* r, double* p, const double* invD,
                 nk_cg_state* st, double* hist, nk_stream_t stream);

/* convergence test on st->rr; else beta (Fletcher-Reeves, or Polak-Ribiere
 * -alpha*zap/rz when flexible) and p = z + beta p with z = invD r (or the
 * explicit z [dev, nullable]).  Records hist[iter] = sqrt(rr). */
int nk_cg_pupdate(int64_t n, const double* r, double* p, const double* invD, const double* z,
                  nk_cg_state* st, double* hist, nk_stream_t stream);

/* ------------------------------------------------------ p-multigrid
 * Building blocks of the Chebyshev-Jacobi p-multigrid preconditioner
 * (V-cycle sequenced by the host, see
 * paper_2104_05829_b200/multigrid.py).  st [nullable]: skip when st->done.
 *
 * Order-to-order transfer, per element (ni, no in [2, 16]):
 *   v   = (in - sub) * wt                    sub, wt nullable
 *   res = (M x M x M) v                      M: no x ni row-major, HOST
 *   res = mask[q] ? res : 0                  mask (output side) nullable
 *   out = accumulate ? out + res : res
 * Restriction: M = J^T with in = r, sub = A e, wt = 1/mult (then gs);
 * prolongation: M = J, accumulate = 1 (J = interp_matrix(coarse -> fine),
 * basis.py:99-117). */
int nk_interp3(int ni, int no, int64_t nelem, const double* M, const double* in,
               const double* sub, const double* wt, const uint8_t* mask, double* out,
               int accumulate, const nk_cg_state* st, nk_stream_t stream);

/* One fused Chebyshev-Jacobi step:
 *   rv = r - Aq (Aq nullable);  res_out = rv (nullable)
 *   d  = a d + b invD rv       (a == 0: d is not read)
 *   e  = (e_acc ? e : 0) + d */
int nk_cheb_step(int64_t n, const double* r, const double* Aq, const double* invD,
                 double* res_out, double* d, double* e, double a, double b, int e_acc,
                 const nk_cg_state* st, nk_stream_t stream);

/* y = A x for a dense row-major n x n A (the explicit inverse of the
 * assembled coarse operator, coarse_solve SPEC.md:519-527). */
int nk_dense_matvec(int64_t n, const double* A, const double* x, double* y,
                    const nk_cg_state* st, nk_stream_t stream);
/* the same with A stored in FP32 (products and sums in FP64): the coarse
 * inverse of the 32-bit smoothing mode, half the streamed bytes.  Row pitch
 * lda >= n, a multiple of 4, with A's columns n..lda-1 zero and x holding lda
 * finite entries; A and x 16-byte aligned. */
int nk_dense_matvec32(int64_t n, int64_t lda, const float* A, const double* x, double* y,
                      const nk_cg_state* st, nk_stream_t stream);

/* inner->done = 1 when outer->done: a nested solve (the iterative coarse
 * solve inside a p-multigrid preconditioner) becomes a no-op once the outer
 * PCG has converged, so graph replays past convergence cost nothing. */
int nk_cg_gate(nk_cg_state* inner, const nk_cg_state* outer, nk_stream_t stream);

/* out[0] = <a, b>_wt (wt nullable = unweighted), deterministic two-stage. */
int nk_wdot(int64_t n, const double* a, const double* b, const double* wt, double* out,
            double* partials, nk_stream_t stream);

/* y = alpha * a * b (* mask when non-null), pointwise -- apply_mass (B u,
 * SPEC.md:380-388) and the Jacobi preconditioner z = invD r
 * outside the fused PCG.  y may alias a or b. */
int nk_pointwise(int64_t n, const double* a, const double* b, double* y, double alpha,
                 const uint8_t* mask, nk_stream_t stream);

/* ---- projection-based initial guesses ----
 * The ProjectionSpace holds k <= NK_PROJ_MAX prior solutions X[q] and A X[q]
 * (row q at X + q*ldx).  project_guess / update are sequenced on the host
 * (paper_2104_05829_b200/projection.py) from these three primitives. */
#define NK_PROJ_MAX 16

/* partial-sum scratch (doubles) nk_multi_wdot needs */
int64_t nk_multi_wdot_partials_len(void);

/* out[q] = sum_i wt_i X[q]_i y_i for q < k (wt nullable), deterministic
 * two-stage reduction; out is [dev] k doubles. */
int nk_multi_wdot(int64_t n, int k, const double* X, int64_t ldx, const double* y,
                  const double* wt, double* out, double* partials, nk_stream_t stream);

/* yout = yin + scale * sum_{q<k} c[q] V[q]   (c [dev] k doubles; yin nullable
 * = 0; yin may alias yout). */
int nk_multi_axpy(int64_t n, int k, const double* c, double scale, const double* V, int64_t ldv,
                  const double* yin, double* yout, nk_stream_t stream);

/* y = x / sqrt(s[0])  (s [dev]); A-normalisation of a new basis vector. */
int nk_vscale(int64_t n, const double* x, double* y, const double* s, nk_stream_t stream);

/* ---- overlapping Schwarz smoother with FDM local solves ----------------
 * (SPEC.md:410-418 fdm_local_solve, 499-507 schwarz_smooth; PAPER.md:228-231,
 * 298-313).  Extended element boxes have (N+3)^3 points [e][k'][j'][i'].
 *   fmap [dev] int32 [E][6][(N+1)^2]: local index (into r) of the point one
 *        layer inside the face neighbour, faces x- x+ y- y+ z- z+, tangential
 *        (slow, fast) = (k,j) | (k,i) | (j,i); -1 = no neighbour.
 *   S    [dev] FP64 [E][3][N+3][N+3]: per element and direction, S[p][mode]
 *        with S^T M S = I (generalised eigenvectors of the 1-D surrogate).
 *   lam  [dev] FP64 [E][3][N+3]: eigenvalues, +inf for dropped points. */

/* out = FDM solve of the extended residual of (r - sub): (S3) diag(1/(lam0
 * (Lx+Ly+Lz) + lam1)) (S3)^T r_ext per element.  out_ext != 0: out is the
 * extended field [E][(N+3)^3] (ASM); else the own points [E][(N+1)^3] (RAS).
 * sub, res_out nullable; res_out (own points) receives r - sub and must not
 * alias r or sub.  fmap entries <= -2 read rx[-src - 2] (values already
 * r - sub received from the neighbour rank; rx nullable when there are
 * none).  Skipped once st->done (st nullable). */
int nk_fdm(int N, int64_t nelem, const double* r, const double* sub, const double* rx,
           double* res_out, const int32_t* fmap, const double* S, const double* lam,
           double lam0, double lam1, double* out, int out_ext, const nk_cg_state* st,
           nk_stream_t stream);

/* nk_fdm with the local solves in FP32 (the paper's 32-bit smoothing,
 * PAPER.md:323-325): r, sub, res_out, out stay FP64; S and lam are FP32
 * copies ([E][3][N+3][N+3], [E][3][N+3]). */
int nk_fdm32(int N, int64_t nelem, const double* r, const double* sub, const double* rx,
             double* res_out, const int32_t* fmap, const float* S, const float* lam,
             double lam0, double lam1, double* out, int out_ext, const nk_cg_state* st,
             nk_stream_t stream);

/* out[i] = a[idx[i]] - b[idx[i]] (b nullable): packs the face-inward layer
 * (r - A e) a neighbour rank's extended boxes need (multi-rank Schwarz). */
int nk_gather_diff(int64_t n, const int32_t* idx, const double* a, const double* b,
                   double* out, const nk_cg_state* st, nk_stream_t stream);

/* z = mask * W * src (own points; src extended [E][(N+3)^3] if src_ext) fused
 * with d = a d + b z (d nullable: d := b z not stored) and e = (e_acc ? e : 0)
 * + d.  W, mask nullable. */
int nk_schwarz_post(int N, int64_t nelem, const double* src, int src_ext, const double* W,
                    const uint8_t* mask, double* d, double* e, double a, double b, int e_acc,
                    const nk_cg_state* st, nk_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* NEKB200_H */
