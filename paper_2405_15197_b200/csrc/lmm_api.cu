// lmm_api.cu -- the C-ABI of liblmm (include/lmm.h): context, memory, call sequencing.
#include <cstdio>
#include <cstring>
#include <new>

#include "lmm_internal.h"

int dev_alloc(DevBuf &b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.p && b.bytes >= bytes) return LMM_OK;
  if (b.p) { cudaFree(b.p); b.p = nullptr; b.bytes = 0; }
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) { cudaGetLastError(); b.p = nullptr; return LMM_E_OOM; }
  b.bytes = bytes;
  return LMM_OK;
}

void dev_free(DevBuf &b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

static cudaEvent_t ev_get(lmm_ctx *c) {
  if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Records an event pair around the outermost timed scope on the context stream; the
// pairs are resolved (synchronised) only when lmm_kernel_times is called.
KTimer::KTimer(lmm_ctx *c_, int cls_) : c(c_), cls(cls_) {
  if (c->timing && c->timer_depth++ == 0) {
    active = true;
    a = ev_get(c);
    cudaEventRecord(a, c->stream);
  }
}
KTimer::~KTimer() {
  if (!c->timing) return;
  c->timer_depth--;
  if (!active) return;
  cudaEvent_t b = ev_get(c);
  cudaEventRecord(b, c->stream);
  c->ev_pending.push_back({cls, a, b});
}

static void resolve_timers(lmm_ctx *c) {
  for (auto &p : c->ev_pending) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    c->k_ms[p.cls] += ms;
    c->k_launch[p.cls] += 1;
    c->ev_pool.push_back(p.a);
    c->ev_pool.push_back(p.b);
  }
  c->ev_pending.clear();
}

// Slab arrays: regular slots K off + K0 n for (off, n) < (2S, N), then the overflow reserve of
// roff virtual CSR entries and rn virtual nodes (spill.cu).  Growing with preserve keeps the
// regular region (the bucketed nodes' results); the overflow region is refilled by the caller.
int slabs_alloc(lmm_ctx *c, int64_t roff, int64_t rn, bool preserve) {
  const int64_t S2 = 2 * c->S, N = c->N;
  // emit records address a node's arc slab as 3 off + 2 n in 32 bits (lmm_load_lattice bound)
  const int64_t lim = (1ll << 32) - 1 - (3 * S2 + 2 * N);
  if (lim <= 0) return LMM_E_ARG;
  if (3 * roff + 2 * rn > lim) { roff = lim / 6; rn = lim / 4; }
  struct Slab { DevBuf *b; size_t rec; int k, k0; };
  const Slab sl[] = {{&c->vert, sizeof(float4), SLAB_V_K, SLAB_V_K0}, {&c->arc, sizeof(ArcRec), SLAB_A_K, SLAB_A_K0},
                     {&c->loop, sizeof(LoopRec), SLAB_L_K, SLAB_L_K0}, {&c->hole_hdr, sizeof(int2), SLAB_H_K, SLAB_H_K0},
                     {&c->hole_ent, sizeof(HoleEnt), SLAB_HE_K, SLAB_HE_K0}};
  for (const Slab &q : sl) {
    const size_t bytes = q.rec * (size_t)(q.k * (S2 + roff) + q.k0 * (N + rn) + 1);
    if (preserve && q.b->p && q.b->bytes < bytes) {
      DevBuf nb;
      int rc;
      if ((rc = dev_alloc(nb, bytes))) return rc;
      CUDA_TRY(cudaMemcpyAsync(nb.p, q.b->p, q.rec * (size_t)(q.k * S2 + q.k0 * N), cudaMemcpyDeviceToDevice, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      dev_free(*q.b);
      *q.b = nb;
    } else {
      int rc;
      if ((rc = dev_alloc(*q.b, bytes))) return rc;
    }
  }
  int rc;
  if ((rc = dev_alloc(c->vmask_hi, sizeof(uint32_t) * (size_t)(SLAB_V_K * roff + SLAB_V_K0 * rn + 1)))) return rc;
  c->ovf_off = roff;
  c->ovf_n = rn;
  return LMM_OK;
}

extern "C" {

LMM_API const char *lmm_version(void) { return "liblmm 0.1 (sm_100a)"; }

LMM_API const char *lmm_error_string(int st) {
  switch (st) {
    case LMM_OK: return "ok";
    case LMM_E_ARG: return "invalid argument";
    case LMM_E_CUDA: return "CUDA error or no usable sm_100 device";
    case LMM_E_OOM: return "device out of memory";
    case LMM_E_STATE: return "call out of order";
    case LMM_E_RADIUS: return "strut end radii disagree with the nodal sphere radius";
    case LMM_E_RANGE: return "triangle range out of bounds";
    default: return "unknown status";
  }
}

LMM_API int lmm_create(lmm_ctx **out, int device, void *stream) {
  if (!out) return LMM_E_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) { cudaGetLastError(); return LMM_E_CUDA; }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return LMM_E_CUDA;
  if (prop.major != 10) return LMM_E_CUDA;   // built for sm_100a only
  if (cudaSetDevice(device) != cudaSuccess) return LMM_E_CUDA;
  lmm_ctx *c = new (std::nothrow) lmm_ctx();
  if (!c) return LMM_E_OOM;
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->n_sm = prop.multiProcessorCount;
  *out = c;
  return LMM_OK;
}

static void free_all(lmm_ctx *c) {
  DevBuf *bufs[] = {&c->node, &c->ends, &c->csr_off, &c->csr_ent, &c->csr_tmp, &c->strut_csr, &c->deg_hist, &c->bucket_nodes,
                    &c->bucket_cnt, &c->node_hdr, &c->vert, &c->arc, &c->loop_hdr, &c->loop, &c->hole_hdr,
                    &c->hole_ent, &c->band, &c->strut_off, &c->node_hole0, &c->node_hole0_64, &c->hole_M,
                    &c->hole_off, &c->hole_bp, &c->hole_node, &c->node_mask, &c->strut_mask, &c->mbits, &c->macc, &c->cmap, &c->brec, &c->ring_n, &c->tmp64, &c->scratch, &c->mm_side, &c->mm_state, &c->tri3, &c->scan_tmp,
                    &c->skey, &c->vmask_hi, &c->spill_list, &c->spill_ctl, &c->spill_ws};
  for (DevBuf *b : bufs) dev_free(*b);
  for (int i = 0; i < LMM_NSTAGE; i++) dev_free(c->stage[i]);
}

LMM_API void lmm_destroy(lmm_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream); else cudaDeviceSynchronize();
  for (int i = 0; i < LMM_NSTAGE; i++)
    if (c->copy_stream[i]) cudaStreamSynchronize(c->copy_stream[i]);
  free_all(c);
  for (int i = 0; i < 2; i++)
    if (c->pinned[i]) cudaFreeHost(c->pinned[i]);
  for (int i = 0; i < LMM_NSTAGE; i++) {
    if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
    if (c->emit_ev[i]) cudaEventDestroy(c->emit_ev[i]);
  }
  for (int i = 0; i < LMM_NSTAGE; i++)
    if (c->copy_stream[i]) cudaStreamDestroy(c->copy_stream[i]);
  resolve_timers(c);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->pinned_scalar) cudaFreeHost(c->pinned_scalar);
  if (c->pinned_hist) cudaFreeHost(c->pinned_hist);
  delete c;
}

LMM_API int lmm_sync(lmm_ctx *c) {
  if (!c) return LMM_E_ARG;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return LMM_OK;
}

LMM_API int lmm_load_lattice(lmm_ctx *c, const float *xyz, int64_t n_nodes, const int64_t *ends, const float *r_end,
                             int64_t n_struts, int where) {
  if (!c || n_nodes < 0 || n_struts < 0 || n_nodes >= (1ll << 31) - 2 || 2 * n_struts >= (1ll << 31) - 2) return LMM_E_ARG;
  // per-band emit records address a node's arc slab as 3 off + 2 n in 32 bits
  if (3 * (2 * n_struts) + 2 * n_nodes >= (1ll << 32)) return LMM_E_ARG;
  if ((n_nodes && !xyz) || (n_struts && (!ends || !r_end))) return LMM_E_ARG;
  if (where != LMM_HOST && where != LMM_DEVICE) return LMM_E_ARG;
  CUDA_TRY(cudaSetDevice(c->device));
  c->lattice_ok = c->mm_ok = c->tri_ok = false;
  c->N = n_nodes;
  c->S = n_struts;
  const float *dx = xyz;
  const int64_t *de = ends;
  const float *dr = r_end;
  void *tmp = nullptr;
  if (where == LMM_HOST) {
    size_t bx = sizeof(float) * 3 * n_nodes, be = sizeof(int64_t) * 2 * n_struts, br = sizeof(float) * 2 * n_struts;
    if (cudaMallocAsync(&tmp, bx + be + br + 64, c->stream) != cudaSuccess) return LMM_E_OOM;
    char *p = (char *)tmp;
    de = (const int64_t *)p;
    dx = (const float *)(p + be);
    dr = (const float *)(p + be + bx);
    // every exit below frees the staging copy (stream-ordered after the copies)
    cudaError_t e = cudaSuccess;
    if (n_struts && e == cudaSuccess) e = cudaMemcpyAsync((void *)de, ends, be, cudaMemcpyHostToDevice, c->stream);
    if (n_nodes && e == cudaSuccess) e = cudaMemcpyAsync((void *)dx, xyz, bx, cudaMemcpyHostToDevice, c->stream);
    if (n_struts && e == cudaSuccess) e = cudaMemcpyAsync((void *)dr, r_end, br, cudaMemcpyHostToDevice, c->stream);
    if (e != cudaSuccess) {
      cudaFreeAsync(tmp, c->stream);
      cudaStreamSynchronize(c->stream);
      return LMM_E_CUDA;
    }
  }
  c->has_node_mask = c->has_strut_mask = false;
  int rc = lattice_build(c, dx, de, dr);
  if (tmp) cudaFreeAsync(tmp, c->stream);
  if (rc) { cudaStreamSynchronize(c->stream); return rc; }
  c->lattice_ok = true;
  return LMM_OK;
}

LMM_API int lmm_build_metamesh(lmm_ctx *c) {
  if (!c) return LMM_E_ARG;
  if (!c->lattice_ok) return LMM_E_STATE;
  CUDA_TRY(cudaSetDevice(c->device));
  c->mm_ok = c->tri_ok = false;
  const int64_t N = c->N, S2 = 2 * c->S;
  int rc;
  if ((rc = degree_buckets(c))) return rc;
  if ((rc = dev_alloc(c->node_hdr, sizeof(int4) * (N + 1)))) return rc;
  if ((rc = dev_alloc(c->loop_hdr, sizeof(int2) * (S2 + 1)))) return rc;
  // overflow reserve for the spilled nodes' virtual slab slots: ~0.2 % of the regular slabs
  if ((rc = slabs_alloc(c, S2 / 512 + 1024, N / 512 + 64, false))) return rc;
  if ((rc = slab_key_init(c))) return rc;
  if ((rc = metamesh_run(c))) return rc;
  if ((rc = spill_run(c))) return rc;
  c->mm_ok = true;
  return LMM_OK;
}

LMM_API int lmm_metamesh_stats(lmm_ctx *c, lmm_stats *out) {
  if (!c || !out) return LMM_E_ARG;
  if (!c->mm_ok) return LMM_E_STATE;
  memset(out, 0, sizeof(*out));
  out->n_nodes = c->N;
  out->n_struts = c->S;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  unsigned long long h[33];
  CUDA_TRY(cudaMemcpy(h, c->deg_hist.p, sizeof(h), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 33; i++) out->degree_hist[i] = (int64_t)h[i];
  // totals from the node headers (host reduction of a copy: introspection only)
  int4 *hdr = (int4 *)malloc(sizeof(int4) * (c->N + 1));
  if (!hdr) return LMM_E_OOM;
  if (c->N) CUDA_TRY(cudaMemcpy(hdr, c->node_hdr.p, sizeof(int4) * c->N, cudaMemcpyDeviceToHost));
  for (int64_t n = 0; n < c->N; n++) {
    int st = hdr[n].x & 0xff;
    out->err_hist[st < LMM_NODE_NCODES ? st : 0]++;
    if (st) { out->n_error_nodes++; continue; }
    out->n_vertices += hdr[n].y & 0xffff;
    out->n_arcs += (hdr[n].y >> 16) & 0xffff;
    out->n_holes += hdr[n].z & 0xffff;
    out->n_loop_entries += (hdr[n].z >> 16) & 0xffff;
    out->n_circular_arcs += hdr[n].w;   // hole entries = cap arcs
  }
  out->n_elliptical_arcs = out->n_arcs - out->n_circular_arcs;
  out->n_spilled_nodes = c->n_spill;
  free(hdr);
  return LMM_OK;
}

LMM_API int lmm_set_emit_mask(lmm_ctx *c, const uint8_t *node_mask, const uint8_t *strut_mask, int where) {
  if (!c || (where != LMM_HOST && where != LMM_DEVICE)) return LMM_E_ARG;
  if (!c->lattice_ok) return LMM_E_STATE;
  CUDA_TRY(cudaSetDevice(c->device));
  const cudaMemcpyKind kind = where == LMM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  int rc;
  c->has_node_mask = node_mask != nullptr;
  c->has_strut_mask = strut_mask != nullptr;
  if (node_mask && c->N) {
    if ((rc = dev_alloc(c->node_mask, (size_t)c->N))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->node_mask.p, node_mask, (size_t)c->N, kind, c->stream));
  }
  if (strut_mask && c->S) {
    if ((rc = dev_alloc(c->strut_mask, (size_t)c->S))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->strut_mask.p, strut_mask, (size_t)c->S, kind, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->tri_ok = false;
  return LMM_OK;
}

LMM_API int lmm_triangulate(lmm_ctx *c, double ce, int64_t *n_tri) {
  // CE >= 1e-8: an arc's subdivision count N (< 2 pi / theta0 + 1) fits the 15 bits of the
  // loop entry (theta0 = 2 acos(1 - CE) > 2 pi / 32767 for CE > 4.6e-9)
  if (!c || !(ce >= 1e-8) || !(ce <= 1.0)) return LMM_E_ARG;
  if (!c->mm_ok) return LMM_E_STATE;
  CUDA_TRY(cudaSetDevice(c->device));
  c->tri_ok = false;
  c->ce = ce;
  c->th0 = (float)(2.0 * acos(1.0 - ce));   // Eq. 11 denominator, once in binary64
  int rc = triangulate_count(c);
  if (rc) return rc;
  c->tri_ok = true;
  if (n_tri) *n_tri = c->n_tri;
  return LMM_OK;
}

LMM_API int lmm_write_triangles(lmm_ctx *c, int64_t first, int64_t count, void *out, int where) {
  if (!c || !out || first < 0 || count < 0) return LMM_E_ARG;
  if (!c->tri_ok) return LMM_E_STATE;
  if (first + count > c->n_tri) return LMM_E_RANGE;
  CUDA_TRY(cudaSetDevice(c->device));
  if (where == LMM_DEVICE) {
    if (((uintptr_t)out) & 15) return LMM_E_ARG;
    return triangulate_emit(c, first, count, out, c->stream);
  }
  if (where != LMM_HOST) return LMM_E_ARG;
  // host destination: emit chunks into two device staging buffers on the context stream
  // and DMA each to the caller's memory on a copy stream, so the copy of chunk b overlaps
  // the emission of chunk b + 1
#ifndef LMM_STAGE_LOG2
#define LMM_STAGE_LOG2 22
#endif
  const int64_t CH = 1ll << LMM_STAGE_LOG2;   // triangles per chunk (2^22: 200 MiB)
  int rc;
  for (int i = 0; i < LMM_NSTAGE; i++) {
    if ((rc = dev_alloc(c->stage[i], (size_t)CH * 50))) return rc;
    if (!c->stage_ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming));
    if (!c->emit_ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->emit_ev[i], cudaEventDisableTiming));
    if (!c->copy_stream[i]) CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream[i], cudaStreamNonBlocking));
  }
  unsigned char *dst = (unsigned char *)out;
  int b = 0;
  bool used[LMM_NSTAGE] = {};
  rc = LMM_OK;
  for (int64_t t = 0; t < count && rc == LMM_OK; t += CH, b = b + 1 == LMM_NSTAGE ? 0 : b + 1) {
    int64_t n = count - t < CH ? count - t : CH;
    // buffer b copied out before it is refilled
    if (used[b] && cudaStreamWaitEvent(c->stream, c->stage_ev[b], 0) != cudaSuccess) { rc = LMM_E_CUDA; break; }
    if ((rc = triangulate_emit(c, first + t, n, c->stage[b].p, c->stream))) break;
    if (cudaEventRecord(c->emit_ev[b], c->stream) != cudaSuccess ||
        cudaStreamWaitEvent(c->copy_stream[b], c->emit_ev[b], 0) != cudaSuccess ||
        cudaMemcpyAsync(dst + t * 50, c->stage[b].p, (size_t)n * 50, cudaMemcpyDeviceToHost, c->copy_stream[b]) != cudaSuccess ||
        cudaEventRecord(c->stage_ev[b], c->copy_stream[b]) != cudaSuccess) { rc = LMM_E_CUDA; break; }
    used[b] = true;
  }
  // on every exit no copy may still be writing into the caller's buffer
  for (int i = 0; i < LMM_NSTAGE; i++)
    if (cudaStreamSynchronize(c->copy_stream[i]) != cudaSuccess && rc == LMM_OK) rc = LMM_E_CUDA;
  if (cudaStreamSynchronize(c->stream) != cudaSuccess && rc == LMM_OK) rc = LMM_E_CUDA;
  return rc;
}

static DevBuf *buf_of(lmm_ctx *c, int id, size_t *bytes) {
  const int64_t N = c->N, S = c->S, S2 = 2 * S;
  DevBuf *b = nullptr;
  size_t n = 0;
  switch (id) {
    case LMM_BUF_CSR_OFF: b = &c->csr_off; n = sizeof(int) * (N + 1); break;
    case LMM_BUF_CSR_ENT: b = &c->csr_ent; n = sizeof(int2) * S2; break;
    case LMM_BUF_NODE_HDR: b = &c->node_hdr; n = sizeof(int4) * N; break;
    case LMM_BUF_VERT: b = &c->vert; n = sizeof(float4) * (SLAB_V_K * (S2 + c->ovf_off) + SLAB_V_K0 * (N + c->ovf_n)); break;
    case LMM_BUF_ARC: b = &c->arc; n = sizeof(ArcRec) * (SLAB_A_K * (S2 + c->ovf_off) + SLAB_A_K0 * (N + c->ovf_n)); break;
    case LMM_BUF_LOOP_HDR: b = &c->loop_hdr; n = sizeof(int2) * S2; break;
    case LMM_BUF_LOOP_ENT: b = &c->loop; n = sizeof(LoopRec) * (SLAB_L_K * (S2 + c->ovf_off) + SLAB_L_K0 * (N + c->ovf_n)); break;
    case LMM_BUF_HOLE_HDR: b = &c->hole_hdr; n = sizeof(int2) * (SLAB_H_K * (S2 + c->ovf_off) + SLAB_H_K0 * (N + c->ovf_n)); break;
    case LMM_BUF_HOLE_ENT: b = &c->hole_ent; n = sizeof(HoleEnt) * (SLAB_HE_K * (S2 + c->ovf_off) + SLAB_HE_K0 * (N + c->ovf_n)); break;
    case LMM_BUF_BAND: b = &c->band; n = sizeof(int4) * S; break;
    case LMM_BUF_STRUT_OFF: b = &c->strut_off; n = sizeof(int64_t) * (S + 1); break;
    case LMM_BUF_HOLE_M: b = &c->hole_M; n = sizeof(int) * c->H; break;
    case LMM_BUF_HOLE_OFF: b = &c->hole_off; n = sizeof(int64_t) * (c->H + 1); break;
    case LMM_BUF_HOLE_BP: b = &c->hole_bp; n = sizeof(float4) * c->H; break;
    case LMM_BUF_NODE_HOLE0: b = &c->node_hole0_64; n = sizeof(int64_t) * (N + 1); break;
    case LMM_BUF_SLAB_KEY: b = &c->skey; n = sizeof(int2) * N; break;
    case LMM_BUF_VMASK_HI: b = &c->vmask_hi; n = sizeof(uint32_t) * (SLAB_V_K * c->ovf_off + SLAB_V_K0 * c->ovf_n); break;
    default: return nullptr;
  }
  if (!b->p) n = 0;
  *bytes = n;
  return b;
}

LMM_API int lmm_buffer_size(lmm_ctx *c, int id, int64_t *bytes) {
  if (!c || !bytes) return LMM_E_ARG;
  size_t n = 0;
  if (!buf_of(c, id, &n)) return LMM_E_ARG;
  *bytes = (int64_t)n;
  return LMM_OK;
}

LMM_API int lmm_copy_buffer(lmm_ctx *c, int id, int64_t offset, int64_t bytes, void *dst) {
  if (!c || !dst || offset < 0 || bytes < 0) return LMM_E_ARG;
  size_t n = 0;
  DevBuf *b = buf_of(c, id, &n);
  if (!b) return LMM_E_ARG;
  if ((size_t)(offset + bytes) > n) return LMM_E_RANGE;
  if (bytes == 0) return LMM_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaMemcpy(dst, (char *)b->p + offset, (size_t)bytes, cudaMemcpyDeviceToHost));
  return LMM_OK;
}

LMM_API int lmm_timing(lmm_ctx *c, int enable) {
  if (!c) return LMM_E_ARG;
  c->timing = enable != 0;
  return LMM_OK;
}

LMM_API int lmm_kernel_times(lmm_ctx *c, double *ms, int64_t *launches) {
  if (!c) return LMM_E_ARG;
  resolve_timers(c);
  for (int i = 0; i < LMM_K_NCLASSES; i++) {
    if (ms) ms[i] = c->k_ms[i];
    if (launches) launches[i] = c->k_launch[i];
  }
  return LMM_OK;
}

LMM_API int lmm_reset_kernel_times(lmm_ctx *c) {
  if (!c) return LMM_E_ARG;
  resolve_timers(c);
  for (int i = 0; i < LMM_K_NCLASSES; i++) { c->k_ms[i] = 0; c->k_launch[i] = 0; }
  return LMM_OK;
}

LMM_API int lmm_launch_count(lmm_ctx *c, int64_t *n) {
  if (!c || !n) return LMM_E_ARG;
  *n = c->n_launch;
  return LMM_OK;
}

LMM_API int lmm_emit_path(lmm_ctx *c, int *path) {
  if (!c || !path) return LMM_E_ARG;
  *path = c->emit_path;
  return LMM_OK;
}

}  // extern "C"
