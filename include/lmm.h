/*
 * lmm.h -- C-ABI of the B200-native lattice meta-meshing library (liblmm.so).
 *
 * The calls follow the paper's problem statement (Zou & Gao, PAPER.md):
 *   load a lattice (node positions, strut index pairs, per-end radii)
 *     -- Sec. 4.3.1 "a strut S_i is defined by its two end vertices v_i^0, v_i^1 and
 *        the corresponding radii r_i^0, r_i^1";
 *   build the meta-mesh (vertices, circular/elliptical arcs, strut and hole faces)
 *     -- Sec. 4.1 definition, Sec. 4.3.1 Eq. 7-9;
 *   triangulate at chord error CE (count pass + prefix scan)
 *     -- Sec. 5 Eq. 11-13, Algorithm 1;
 *   write triangles as binary-STL records
 *     -- Sec. 1 "transform them into the STL format".
 *
 * Conventions
 *  - Every call returns an lmm_status (LMM_OK = 0); lmm_error_string() names it.
 *    A call that fails leaves the context usable; nothing ever falls back to a CPU
 *    implementation: a missing/unsupported CUDA device is LMM_E_CUDA.
 *  - `where` arguments say whether a pointer is host memory (LMM_HOST) or device
 *    memory of the context's device (LMM_DEVICE).  Caller-owned buffers stay owned by
 *    the caller; the library only reads inputs during the call and only writes outputs
 *    inside [out, out + bytes).  All library memory is owned by the context and freed by
 *    lmm_destroy().
 *  - Work is enqueued on the CUDA stream given to lmm_create (NULL = legacy default
 *    stream).  Calls that return sizes synchronise that stream; lmm_write_triangles
 *    with a device destination is asynchronous (call lmm_sync before reading).
 *  - Node indices are 0-based int64 in the API and must be < 2^31 (internal int32).
 *  - Geometry is binary32, topology decisions follow the fixed-order binary32 spec of
 *    DESIGN.md Sec. 4 (bit-identical to the CPU oracle's decisions).
 */
#ifndef LMM_H
#define LMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMM_API __attribute__((visibility("default")))

typedef enum {
  LMM_OK = 0,
  LMM_E_ARG = 1,         /* invalid argument (null pointer, negative size, bad index)  */
  LMM_E_CUDA = 2,        /* CUDA runtime error or no usable sm_100 device              */
  LMM_E_OOM = 3,         /* device allocation failed                                   */
  LMM_E_STATE = 4,       /* call out of order (e.g. triangulate before build)          */
  LMM_E_RADIUS = 5,      /* struts meeting at a node disagree on that node's radius     */
  LMM_E_RANGE = 6        /* requested triangle range outside [0, n_triangles)          */
} lmm_status;

enum { LMM_HOST = 0, LMM_DEVICE = 1 };

/* Per-node meta-mesh status codes (lmm_stats.err_hist index); identical meanings to
 * the oracle's ORC_E_* codes.  DEGREE = degree > 63.  JCAP/CCAP/ACAP/QCAP mark a bucket
 * workspace exceeded inside lmm_build_metamesh; such nodes are meta-meshed again by the spill
 * kernel, so they are not reported afterwards (ACAP would remain only for a node of more than
 * 1023 vertices, which degree <= 63 cannot reach).  CHAIN/HOLE/ANGLE/UNREF/EMPTY are reported
 * only if the topology closes at no vertex resolution delta_c * 2^level, level 0..4. */
enum {
  LMM_NODE_OK = 0, LMM_NODE_DEGREE = 1, LMM_NODE_STRUT = 2, LMM_NODE_JCAP = 3,
  LMM_NODE_CCAP = 4, LMM_NODE_ACAP = 5, LMM_NODE_CONIC = 6, LMM_NODE_UNREF = 7,
  LMM_NODE_CHAIN = 8, LMM_NODE_ANGLE = 9, LMM_NODE_EMPTY = 10, LMM_NODE_HOLE = 11,
  LMM_NODE_SHORT = 12, LMM_NODE_QCAP = 13, LMM_NODE_NCODES = 14
};

typedef struct lmm_ctx lmm_ctx;

typedef struct {
  int64_t n_nodes, n_struts;
  int64_t n_vertices, n_arcs, n_elliptical_arcs, n_circular_arcs;
  int64_t n_loop_entries, n_holes;
  int64_t n_error_nodes;
  int64_t err_hist[LMM_NODE_NCODES];
  int64_t degree_hist[33];  /* nodes by degree 0..31, [32] = degree > 31 */
  int64_t n_spilled_nodes;  /* nodes meta-meshed by the spill kernel (degree 32..63, a bucket
                               workspace exceeded, or re-decided at a coarser resolution) */
} lmm_stats;

/* Create a context on CUDA device `device`, enqueuing on `cuda_stream`
 * (a cudaStream_t, may be NULL).  *out receives the context. */
LMM_API int lmm_create(lmm_ctx **out, int device, void *cuda_stream);

/* Free every device buffer owned by the context. */
LMM_API void lmm_destroy(lmm_ctx *ctx);

/* Load a lattice (replaces any previous one).
 *   xyz   : float32 [n_nodes][3] node centres v (row-major)
 *   ends  : int64   [n_struts][2] strut endpoint node indices (i0, i1), i0 != i1
 *   r_end : float32 [n_struts][2] strut radius at i0 and at i1; struts are tangent to the
 *           nodal spheres (Sec. 4.1), so every strut end at a node must carry
 *           that node's sphere radius (else LMM_E_RADIUS); radii > 0.
 *   where : LMM_HOST or LMM_DEVICE for all three arrays.
 * Sizes: n_nodes < 2^31 - 2, 2 n_struts < 2^31 - 2 and 6 n_struts + 2 n_nodes < 2^32 (one
 * context holds up to ~700M struts; device memory is the binding limit well before that),
 * else LMM_E_ARG.
 * Builds the device CSR (node -> incident struts, ascending strut id). */
LMM_API int lmm_load_lattice(lmm_ctx *ctx, const float *xyz, int64_t n_nodes,
                             const int64_t *ends, const float *r_end, int64_t n_struts,
                             int where);

/* Build the meta-mesh of every node: degree histogram + degree-bucketed schedule,
 * then the per-node kernels (sides, triple junctions, vertex clusters, arcs via Eq. 7,
 * arc loops per strut end, hole contours): lane groups per node for degree <= 31, a CTA
 * per node (spill kernel) for degree 32..63, for nodes that exceed their bucket's
 * workspace and for nodes re-decided at a coarser vertex resolution (R10).
 * Nodes the model cannot represent (degree > 63, a strut too short or degenerate, an
 * unbounded conic carrying a vertex, a topology that does not close at any resolution)
 * get a non-zero status (see lmm_stats); they contribute no triangles. */
LMM_API int lmm_build_metamesh(lmm_ctx *ctx);

/* Totals and histograms of the current meta-mesh (synchronises). */
LMM_API int lmm_metamesh_stats(lmm_ctx *ctx, lmm_stats *out);

/* Restrict emission to a subset (spatial partitioning across GPUs): only struts with
 * strut_mask[s] != 0 contribute their band and only nodes with node_mask[n] != 0 their
 * hole fans (counts become 0 otherwise; the meta-mesh of every node is still built, so
 * halo nodes give the bands of boundary struts their far-end loops).
 *   node_mask  : uint8 [n_nodes] or NULL (= all), strut_mask : uint8 [n_struts] or NULL (= all)
 *   where      : LMM_HOST or LMM_DEVICE for both arrays.
 * Cleared by lmm_load_lattice; takes effect at the next lmm_triangulate. */
LMM_API int lmm_set_emit_mask(lmm_ctx *ctx, const uint8_t *node_mask, const uint8_t *strut_mask, int where);

/* Count pass for chord error CE (fraction of the radius, 0 < CE <= 1): per-arc
 * subdivision counts N (Eq. 11), band and hole triangle counts, device prefix scan of
 * the output offsets.  *n_triangles receives the total (synchronises).  Reuses the
 * meta-mesh: calling it again with another CE re-triangulates without re-meta-meshing
 * (Sec. 5 "we only need to re-subdivide the arcs"). */
LMM_API int lmm_triangulate(lmm_ctx *ctx, double chord_error, int64_t *n_triangles);

/* Emit triangles [first, first + count) of the global order (struts ascending, each
 * strut's band; then nodes ascending, each node's hole fans) as 50-byte binary-STL
 * facet records (normal f32x3, v1, v2, v3 f32x3 each, uint16 attribute = 0), packed, into
 * out[0 .. 50*count).  `out` is host or device memory per `where`; device `out` must be
 * 16-byte aligned.  Host output is staged through pinned buffers in chunks.
 * The band region is emitted by one of two kernels that write identical bytes (DESIGN.md
 * Sec. 6): warp per band when the mean band exceeds 100 triangles, else CTA windows of
 * whole bands; environment overrides for tuning only: LMM_EMIT_PATH=0|1 (band | windows),
 * LMM_SPCW (window points, 256..1280), LMM_SPAN (band triangles per CTA, multiple of 64),
 * LMM_PCAP (band-path point cache, 152 + 16 k below 640, or 640; default from the mean band). */
LMM_API int lmm_write_triangles(lmm_ctx *ctx, int64_t first, int64_t count, void *out, int where);

/* Wait for all work enqueued by the context. */
LMM_API int lmm_sync(lmm_ctx *ctx);

/* ---- introspection (tests, benchmarks) ---------------------------------------------- */

/* Internal buffers, copied out for parity checks.  `id` is one of LMM_BUF_*;
 * lmm_buffer_size gives its size in bytes, lmm_copy_buffer copies `bytes` from `offset`
 * into host memory `dst`.  Layouts are documented in DESIGN.md Sec. 5. */
enum {
  LMM_BUF_CSR_OFF = 0,      /* int32 [N+1]                                            */
  LMM_BUF_CSR_ENT = 1,      /* int32x2 [2S]: strut id, far node | end<<31            */
  LMM_BUF_NODE_HDR = 2,     /* int32x4 [N]: status|d<<8, nv|na<<16, nh|nle<<16, nhe   */
  LMM_BUF_VERT = 3,         /* float32x4 [3*off+2n slab]: x, y, z (node-local), mask  */
  LMM_BUF_ARC = 4,          /* 12 x 32-bit [3*off+2n slab]: lo|hi<<8|vs<<16|ve<<24,    */
                            /*   t0, dt, o.xyz, a.xyz, b.xyz                          */
  LMM_BUF_LOOP_HDR = 5,     /* int32x2 [2S] per CSR entry: first entry (node slab), n */
  LMM_BUF_LOOP_ENT = 6,     /* 4 x 32-bit [6*off+4n slab]: arc|fwd<<16, phs, dph, cum */
  LMM_BUF_HOLE_HDR = 7,     /* int32x2 [off+n slab]: first hole entry, n entries       */
  LMM_BUF_HOLE_ENT = 8,     /* int32 [3*off+2n slab]: arc | fwd<<16                   */
  LMM_BUF_BAND = 9,         /* int32x4 [S]: nA, nB, kB, 0  (after lmm_triangulate)    */
  LMM_BUF_STRUT_OFF = 10,   /* int64 [S+1] triangle offsets of the bands              */
  LMM_BUF_HOLE_M = 11,      /* int32 [H]: triangles per hole (global hole order)      */
  LMM_BUF_HOLE_OFF = 12,    /* int64 [H+1] triangle offsets of the holes (after bands)*/
  LMM_BUF_HOLE_BP = 13,     /* float32x4 [H]: fan centre b_project (node-local), node */
  LMM_BUF_NODE_HOLE0 = 14,  /* int64 [N+1]: global index of each node's first hole     */
  LMM_BUF_SLAB_KEY = 15,    /* int32x2 [N]: slab key (off, n) of each node: its slabs   */
                            /*   start at K off + K0 n (K, K0 per slab above); nodes of */
                            /*   the spill kernel have virtual keys (>= (2S, N)) into   */
                            /*   the overflow reserve behind the regular slots          */
  LMM_BUF_VMASK_HI = 16,    /* uint32 [2 ovf_off + 2 ovf_n]: tie-mask bits 32..63 of the */
                            /*   overflow vertex slots (slab index - (4S + 2N))          */
  LMM_BUF_COUNT = 17
};
LMM_API int lmm_buffer_size(lmm_ctx *ctx, int id, int64_t *bytes);
LMM_API int lmm_copy_buffer(lmm_ctx *ctx, int id, int64_t offset, int64_t bytes, void *dst);

/* Kernel timing (CUDA events around each launch on the context stream).  Enable, run,
 * then read the accumulated milliseconds and launch counts per kernel class
 * (LMM_K_*).  Disabled by default (no events recorded). */
enum {
  LMM_K_CSR = 0, LMM_K_BUCKET = 1, LMM_K_METAMESH = 2, LMM_K_COUNT = 3, LMM_K_SCAN = 4,
  LMM_K_EMIT = 5, LMM_K_NCLASSES = 6
};
LMM_API int lmm_timing(lmm_ctx *ctx, int enable);
LMM_API int lmm_kernel_times(lmm_ctx *ctx, double *ms /*[LMM_K_NCLASSES]*/, int64_t *launches /*[LMM_K_NCLASSES]*/);
LMM_API int lmm_reset_kernel_times(lmm_ctx *ctx);

/* Number of CUDA kernels this context has launched so far (monotone counter). */
LMM_API int lmm_launch_count(lmm_ctx *ctx, int64_t *n);

/* The kernel that emitted the band region in the last lmm_write_triangles: 0 = warp per band
 * (k_emit), 1 = CTA windows of whole bands (k_emit_span), -1 = none yet. */
LMM_API int lmm_emit_path(lmm_ctx *ctx, int *path);

LMM_API const char *lmm_error_string(int status);
LMM_API const char *lmm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LMM_H */
