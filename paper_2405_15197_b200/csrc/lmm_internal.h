// lmm_internal.h -- host-side context and kernel launch interfaces of liblmm.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/lmm.h"
#include "lmm_common.cuh"

#define LMM_NBUCKET 6   // degree buckets 1..4, 5..8, 9..12, 13..16, 17..23, 24..31 (0, >31 apart)

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
};

struct lmm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int n_sm = 148;
  int64_t N = 0, S = 0;
  // lattice
  DevBuf node;       // float4 [N]  x, y, z, r
  DevBuf ends;       // int2   [S]
  DevBuf csr_off;    // int    [N+1]
  DevBuf csr_ent;    // int2   [2S] strut, far | end<<31
  DevBuf strut_csr;  // int2   [S]  CSR entry of the strut at i0 and at i1
  DevBuf csr_tmp;    // int2   [2S] CSR fill before ranking (swapped with csr_ent)
  DevBuf deg_hist;   // unsigned long long [33]
  DevBuf bucket_nodes;   // int [N]
  DevBuf bucket_cnt;     // int [LMM_NBUCKET + 2]
  int64_t bucket_off[LMM_NBUCKET + 3] = {0};
  bool lattice_ok = false;
  // meta-mesh
  DevBuf node_hdr;   // int4 [N]
  DevBuf vert;       // float4 slab
  DevBuf arc;        // ArcRec slab
  DevBuf loop_hdr;   // int2 [2S]
  DevBuf loop;       // LoopRec slab
  DevBuf hole_hdr;   // int2 slab
  DevBuf hole_ent;   // HoleEnt slab
  DevBuf skey;       // int2 [N] slab key (off, n): slab base of node n is K off + K0 n;
                     //   spilled nodes get a virtual key (2S + voff, N + vn) in the overflow reserve
  DevBuf vmask_hi;   // uint32 per overflow vertex slot: tie-mask bits 32..63 (degree > 31)
  int64_t ovf_off = 0, ovf_n = 0;   // overflow reserve behind the regular slabs (virtual CSR entries, nodes)
  DevBuf spill_list; // int [N] nodes for the spill kernel
  DevBuf spill_ctl;  // unsigned long long [8] spill control words
  DevBuf spill_ws;   // per-CTA spill workspace
  int64_t spill_wsb = 0;   // spill workspace bytes per CTA
  int64_t n_spill = 0;     // nodes meta-meshed by the spill kernel in the last build
  bool mm_ok = false;
  // triangulation
  double ce = 0.0;
  float th0 = 0.0f;
  DevBuf band;       // int4 [S] nA, nB, kB, 0
  DevBuf strut_off;  // int64 [S+1]
  DevBuf node_hole0; // int [N+1]  (int64 scan kept in tmp)
  DevBuf node_hole0_64;
  DevBuf hole_M;     // int [H]
  DevBuf hole_off;   // int64 [H+1]
  DevBuf hole_bp;    // float4 [H]
  DevBuf hole_node;  // int [H]
  DevBuf node_mask;  // uint8 [N] hole emission mask (empty = all)
  DevBuf strut_mask; // uint8 [S] band emission mask (empty = all)
  bool has_node_mask = false, has_strut_mask = false;
  DevBuf mbits;      // uint32 merge bits (1 per band triangle)
  DevBuf macc;       // int per merge word
  DevBuf cmap;       // int per emit chunk
  DevBuf brec;       // 64-byte emit record per strut band
  DevBuf ring_n;     // int [2S] points per ring (CSR entry), count pass
  int64_t H = 0, n_tri = 0, n_tri_band = 0;
  bool emit_attr_set = false;   // k_emit's opt-in shared-memory limit set on this context's device
  int emit_occ[64] = {0};       // CTAs per SM: k_emit by point-cache size [0, 32), k_emit_span by window [40, 51)
  int emit_path = -1;           // band region of the last emission: 0 k_emit, 1 k_emit_span
  bool tri_ok = false;
  // scratch
  DevBuf tmp64;      // int64 scan scratch
  DevBuf scratch;    // misc
  DevBuf tri3;       // uint32 lexicographic triple table (meta-mesh junction enumeration)
  DevBuf mm_side;    // float4 [2S][5] side records between the meta-mesh parts
  DevBuf mm_state;   // int4 [N] node state between the meta-mesh parts
  DevBuf scan_tmp;   // scan tile sums (all recursion levels)
  int64_t *pinned_scalar = nullptr;   // pinned host words for scan totals / flags
  unsigned long long *pinned_hist = nullptr;   // pinned degree histogram + bucket bases
#ifndef LMM_NSTAGE
#define LMM_NSTAGE 3      // device staging buffers (and copy streams) of host output
#endif
  DevBuf stage[LMM_NSTAGE];   // device staging for host output
  void *pinned[2] = {nullptr, nullptr};
  size_t pinned_bytes = 0;
  cudaEvent_t stage_ev[LMM_NSTAGE] = {};   // staging buffer b free again (copy done)
  cudaEvent_t emit_ev[LMM_NSTAGE] = {};    // staging buffer b filled (emit done)
  cudaStream_t copy_stream[LMM_NSTAGE] = {};   // device -> host copies of host output (one per staging buffer)
  // timing
  bool timing = false;
  double k_ms[LMM_K_NCLASSES] = {0};
  int64_t k_launch[LMM_K_NCLASSES] = {0};
  struct EvPair { int cls; cudaEvent_t a, b; };
  std::vector<EvPair> ev_pending;
  std::vector<cudaEvent_t> ev_pool;
  int timer_depth = 0;
  int64_t n_launch = 0;   // kernels launched by this context
};

// memory helpers (lmm_api.cu)
int dev_alloc(DevBuf &b, size_t bytes);
void dev_free(DevBuf &b);

// timing scope: records events around a launch when ctx->timing
struct KTimer {
  lmm_ctx *c;
  int cls;
  bool active = false;
  cudaEvent_t a = nullptr;
  KTimer(lmm_ctx *c_, int cls_);
  ~KTimer();
};

// lattice.cu
int lattice_build(lmm_ctx *c, const float *xyz_dev, const int64_t *ends_dev, const float *rend_dev);
int degree_buckets(lmm_ctx *c);
// metamesh.cu
int metamesh_run(lmm_ctx *c);
// spill.cu
int slab_key_init(lmm_ctx *c);
int spill_run(lmm_ctx *c);
// lmm_api.cu: slab arrays with an overflow reserve of roff virtual CSR entries / rn virtual
// nodes; preserve = keep the regular region's contents when growing
int slabs_alloc(lmm_ctx *c, int64_t roff, int64_t rn, bool preserve);
// scan.cu
int scan_exclusive_i64(lmm_ctx *c, const int64_t *in, int64_t *out, int64_t n, int64_t *total_host);
int scan_exclusive_i32_to_i64(lmm_ctx *c, const int *in, int64_t *out, int64_t n, int64_t *total_host);
// triangulate.cu
int triangulate_count(lmm_ctx *c);
int triangulate_emit(lmm_ctx *c, int64_t first, int64_t count, void *out_dev, cudaStream_t st);

#define CUDA_TRY(x)                                   \
  do {                                                \
    cudaError_t e__ = (x);                            \
    if (e__ != cudaSuccess) return LMM_E_CUDA;        \
  } while (0)
