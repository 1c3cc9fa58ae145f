// triangulate.cu -- resolution-parametric triangulation of the meta-mesh
// (Sec. 5: Eq. 11 subdivision counts, Eq. 12 uniform parameters, strut bands
// "by connecting these vertices", Eq. 13 hole fans, Algorithm 1).
//
// Count pass (one thread per strut / per node): N per arc from the chord error, loop
// point counts, the band rotation, hole sizes and fan centres; device scans give the
// output offsets.  Emit pass: output-centric -- each CTA owns a contiguous range of the
// global triangle order, so writes are perfectly balanced and contiguous: triangles are
// assembled as 50-byte STL records in shared memory and leave with one TMA bulk store
// (cp.async.bulk.global.shared::cta) per chunk.
//
// Decision arithmetic (N, stitch keys, band rotation, merge order) is binary32 with the
// operation order of DESIGN.md Sec. 4.5 written with explicit round-to-nearest
// intrinsics (never contracted); geometry uses the fast paths.
#include "lmm_internal.h"

namespace {

struct TriParams {
  const float4 *node;
  const int *csr_off;
  const int2 *ends;
  const int2 *strut_csr;
  const int4 *node_hdr;
  const float4 *vert;
  const ArcRec *arc;
  const int2 *loop_hdr;
  LoopRec *loop;
  const int2 *hole_hdr;
  HoleEnt *hole_ent;
  float th0;
  int64_t S, N;
  int4 *band;
  int64_t *band_cnt;        // [S] nA + nB (scan input)
  const int64_t *strut_off; // [S+1]
  const int64_t *node_hole0;// [N+1]
  int *hole_M;              // [H]
  const int64_t *hole_off;  // [H+1]
  float4 *hole_bp;          // [H]
  int *hole_node;           // [H]
  int64_t H;
  int64_t n_tri_band;
};

__device__ __forceinline__ int arc_N(float dt, float th0) { return (int)floorf(__fdiv_rn(dt, th0)) + 1; }

__device__ __forceinline__ float key_at(float phs, float dph, int N, int j) {
  // phs + j * (dph / N), each operation rounded
  return __fadd_rn(phs, __fmul_rn((float)j, __fdiv_rn(dph, (float)N)));
}

__device__ __forceinline__ float wrap_rel(float b, float a0) {
  float r = __fsub_rn(b, a0);
  if (r < 0.0f) r = __fadd_rn(r, LMM_TWO_PI_F);
  if (r >= LMM_TWO_PI_F) r = __fsub_rn(r, LMM_TWO_PI_F);
  return r;
}

__device__ __forceinline__ int64_t vbase(const int *off, int n) { return slab_base(off[n], n, SLAB_V_K, SLAB_V_K0); }
__device__ __forceinline__ int64_t abase(const int *off, int n) { return slab_base(off[n], n, SLAB_A_K, SLAB_A_K0); }
__device__ __forceinline__ int64_t lbase(const int *off, int n) { return slab_base(off[n], n, SLAB_L_K, SLAB_L_K0); }
__device__ __forceinline__ int64_t hbase(const int *off, int n) { return slab_base(off[n], n, SLAB_H_K, SLAB_H_K0); }
__device__ __forceinline__ int64_t hebase(const int *off, int n) { return slab_base(off[n], n, SLAB_HE_K, SLAB_HE_K0); }

// Eq. 12 point jj of an arc, node-local; the endpoints are the shared vertices exactly
__device__ __forceinline__ f3 arc_point(const ArcRec &A, const float4 *vslab, int N, int jj) {
  if (jj == 0 || jj == N) {
    int v = jj == 0 ? (A.ids >> 16) & 0xff : (A.ids >> 24);
    float4 p = vslab[v];
    return F3(p.x, p.y, p.z);
  }
  float t = A.t0 + (float)jj * (A.dt / (float)N);
  t = t - LMM_TWO_PI_F * rintf(t * (1.0f / LMM_TWO_PI_F));
  float s, c;
  __sincosf(t, &s, &c);
  return F3(fmaf(A.ax, s, fmaf(A.bx, c, A.ox)), fmaf(A.ay, s, fmaf(A.by, c, A.oy)), fmaf(A.az, s, fmaf(A.bz, c, A.oz)));
}

// ---------------------------------------------------------------------------------
// count pass
// ---------------------------------------------------------------------------------
__global__ void k_band_count(TriParams P) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= P.S) return;
  int2 e = P.ends[s];
  int2 ce = P.strut_csr[s];
  int4 hA = P.node_hdr[e.x], hB = P.node_hdr[e.y];
  int nA = 0, nB = 0, kB = 0;
  if ((hA.x & 0xff) == 0 && (hB.x & 0xff) == 0) {
    int2 LA = P.loop_hdr[ce.x], LB = P.loop_hdr[ce.y];
    LoopRec *la = P.loop + lbase(P.csr_off, e.x) + LA.x;
    LoopRec *lb = P.loop + lbase(P.csr_off, e.y) + LB.x;
    const ArcRec *aa = P.arc + abase(P.csr_off, e.x);
    const ArcRec *ab = P.arc + abase(P.csr_off, e.y);
    for (int i = 0; i < LA.y; i++) {
      la[i].cum = nA;
      nA += arc_N(aa[la[i].arc_fwd & 0xffff].dt, P.th0);
    }
    for (int i = 0; i < LB.y; i++) {
      lb[i].cum = nB;
      nB += arc_N(ab[lb[i].arc_fwd & 0xffff].dt, P.th0);
    }
    if (nA > 0 && nB > 0) {
      // rotation of ring B: first point minimising its angle relative to A's start
      float a0 = la[0].phs;
      float best = 0.0f;
      int idx = 0;
      for (int i = 0; i < LB.y; i++) {
        float phs = lb[i].phs, dph = lb[i].dph;
        int N = arc_N(ab[lb[i].arc_fwd & 0xffff].dt, P.th0);
        for (int j = 0; j < N; j++, idx++) {
          float r = wrap_rel(key_at(phs, dph, N, j), a0);
          if (idx == 0 || r < best) { best = r; kB = idx; }
        }
      }
    } else { nA = nB = 0; }
  }
  P.band[s] = make_int4(nA, nB, kB, 0);
  P.band_cnt[s] = (int64_t)nA + nB;
}

__global__ void k_node_nholes(const int4 *hdr, int64_t N, int *nh) {
  int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= N) return;
  int4 h = hdr[n];
  nh[n] = (h.x & 0xff) == 0 ? (h.z & 0xffff) : 0;
}

__global__ void k_hole_count(TriParams P) {
  int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= P.N) return;
  int64_t g0 = P.node_hole0[n], g1 = P.node_hole0[n + 1];
  if (g0 == g1) return;
  const float4 on = P.node[n];
  const float R = on.w;
  const float4 *vs = P.vert + vbase(P.csr_off, (int)n);
  const ArcRec *as = P.arc + abase(P.csr_off, (int)n);
  const int2 *hh = P.hole_hdr + hbase(P.csr_off, (int)n);
  HoleEnt *he = P.hole_ent + hebase(P.csr_off, (int)n);
  for (int64_t g = g0; g < g1; g++) {
    int2 H = hh[g - g0];
    int M = 0;
    for (int i = 0; i < H.y; i++) {
      he[H.x + i].cum = M;
      M += arc_N(as[he[H.x + i].arc_fwd & 0xffff].dt, P.th0);
    }
    // Eq. 13 fan centre: barycentre of the contour vertices, direction regularised by
    // the contour's outward (Newell) normal (reading R7)
    float bx = 0.f, by = 0.f, bz = 0.f, nx = 0.f, ny = 0.f, nz = 0.f;
    f3 first = F3(0.f, 0.f, 0.f), prev = first;
    bool have = false;
    for (int i = 0; i < H.y; i++) {
      uint32_t af = he[H.x + i].arc_fwd;
      const ArcRec A = as[af & 0xffff];
      int fwd = af >> 16;
      int N = arc_N(A.dt, P.th0);
      for (int j = 0; j < N; j++) {
        f3 p = arc_point(A, vs, N, fwd ? j : N - j);
        bx += p.x; by += p.y; bz += p.z;
        if (have) {
          f3 cr = f_cross(prev, p);
          nx += cr.x; ny += cr.y; nz += cr.z;
        } else { first = p; have = true; }
        prev = p;
      }
    }
    {
      f3 cr = f_cross(prev, first);
      nx += cr.x; ny += cr.y; nz += cr.z;
    }
    float inv = 1.0f / (float)M;
    float nl = rsqrtf(nx * nx + ny * ny + nz * nz);
    float dx = bx * inv + R * nx * nl, dy = by * inv + R * ny * nl, dz = bz * inv + R * nz * nl;
    float dl = R * rsqrtf(dx * dx + dy * dy + dz * dz);
    P.hole_M[g] = M;
    P.hole_bp[g] = make_float4(dx * dl, dy * dl, dz * dl, 0.0f);
    P.hole_node[g] = (int)n;
  }
}

// ---------------------------------------------------------------------------------
// emit pass
// ---------------------------------------------------------------------------------
constexpr int EMIT_T = 256;          // threads per CTA
constexpr int EMIT_R = 8;            // consecutive triangles per thread
constexpr int EMIT_TPC = EMIT_T * EMIT_R;   // triangles per chunk (2048 -> 102400 B)
constexpr int REC = 50;

struct Ring {
  const LoopRec *le;
  const ArcRec *arcs;
  const float4 *vs;
  int cnt;
  int n;
  float ox, oy, oz;
};

__device__ __forceinline__ int ring_entry(const Ring &r, int idx) {
  int e = 0;
  while (e + 1 < r.cnt && r.le[e + 1].cum <= idx) e++;
  return e;
}

__device__ __forceinline__ float ring_key(const Ring &r, int idx, float th0) {
  int e = ring_entry(r, idx);
  const LoopRec L = r.le[e];
  int N = arc_N(r.arcs[L.arc_fwd & 0xffff].dt, th0);
  return key_at(L.phs, L.dph, N, idx - L.cum);
}

__device__ __forceinline__ f3 ring_point(const Ring &r, int idx, float th0) {
  int e = ring_entry(r, idx);
  const LoopRec L = r.le[e];
  const ArcRec A = r.arcs[L.arc_fwd & 0xffff];
  int N = arc_N(A.dt, th0);
  int j = idx - L.cum;
  f3 p = arc_point(A, r.vs, N, (L.arc_fwd >> 16) ? j : N - j);
  return F3(r.ox + p.x, r.oy + p.y, r.oz + p.z);
}

__device__ __forceinline__ void put_rec(unsigned char *dst, f3 a, f3 b, f3 c) {
  f3 u = f_sub(b, a), v = f_sub(c, a);
  float nx = u.y * v.z - u.z * v.y, ny = u.z * v.x - u.x * v.z, nz = u.x * v.y - u.y * v.x;
  float l2 = nx * nx + ny * ny + nz * nz;
  float il = l2 > 0.0f ? rsqrtf(l2) : 0.0f;
  float f[12] = {nx * il, ny * il, nz * il, a.x, a.y, a.z, b.x, b.y, b.z, c.x, c.y, c.z};
  uint16_t *d16 = reinterpret_cast<uint16_t *>(dst);   // records are 2-byte aligned
#pragma unroll
  for (int i = 0; i < 12; i++) {
    uint32_t w = __float_as_uint(f[i]);
    d16[2 * i] = (uint16_t)(w & 0xffffu);
    d16[2 * i + 1] = (uint16_t)(w >> 16);
  }
  d16[24] = 0;
}

__device__ __forceinline__ int64_t upper_bound64(const int64_t *a, int64_t lo, int64_t hi, int64_t x) {
  // first index in [lo, hi) with a[i] > x
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (a[m] <= x) lo = m + 1; else hi = m;
  }
  return lo;
}

struct BandState {
  Ring A, B;
  int nA, nB, kB;
  float a0;
  int i, j;
  float an, bn;           // next keys
  f3 pa, pa1, pb, pb1;    // A_i, A_{i+1}, B_j, B_{j+1} (rotated indices)
};

__device__ __forceinline__ float keyA(const BandState &S, int i, float th0) {
  return i < S.nA ? __fsub_rn(ring_key(S.A, i, th0), S.a0) : LMM_TWO_PI_F;
}
__device__ __forceinline__ float keyB(const BandState &S, int j, float th0) {
  if (j < S.nB) return wrap_rel(ring_key(S.B, (j + S.kB) % S.nB, th0), S.a0);
  return __fadd_rn(wrap_rel(ring_key(S.B, S.kB, th0), S.a0), LMM_TWO_PI_F);
}

__device__ void band_open(const TriParams &P, int64_t s, int q, BandState &S) {
  int2 e = P.ends[s];
  int2 ce = P.strut_csr[s];
  int4 bd = P.band[s];
  S.nA = bd.x; S.nB = bd.y; S.kB = bd.z;
  int2 LA = P.loop_hdr[ce.x], LB = P.loop_hdr[ce.y];
  float4 oa = P.node[e.x], ob = P.node[e.y];
  S.A.le = P.loop + lbase(P.csr_off, e.x) + LA.x;
  S.A.arcs = P.arc + abase(P.csr_off, e.x);
  S.A.vs = P.vert + vbase(P.csr_off, e.x);
  S.A.cnt = LA.y; S.A.n = S.nA; S.A.ox = oa.x; S.A.oy = oa.y; S.A.oz = oa.z;
  S.B.le = P.loop + lbase(P.csr_off, e.y) + LB.x;
  S.B.arcs = P.arc + abase(P.csr_off, e.y);
  S.B.vs = P.vert + vbase(P.csr_off, e.y);
  S.B.cnt = LB.y; S.B.n = S.nB; S.B.ox = ob.x; S.B.oy = ob.y; S.B.oz = ob.z;
  S.a0 = S.A.le[0].phs;
  // merge path: smallest i with (j==0 || i==nA || key B_{j} < key A_{i+1}), j = q - i,
  // keys 1-based: A key m = keyA(m) (m = nA -> 2pi), B key m = keyB(m)
  int lo = q - S.nB > 0 ? q - S.nB : 0, hi = q < S.nA ? q : S.nA;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int jj = q - mid;
    bool pr = (jj == 0) || (keyB(S, jj, P.th0) < keyA(S, mid + 1, P.th0));
    if (pr) hi = mid; else lo = mid + 1;
  }
  S.i = lo; S.j = q - lo;
  S.an = keyA(S, S.i + 1, P.th0);
  S.bn = keyB(S, S.j + 1, P.th0);
  S.pa = ring_point(S.A, S.i % S.nA, P.th0);
  S.pa1 = ring_point(S.A, (S.i + 1) % S.nA, P.th0);
  S.pb = ring_point(S.B, (S.j + S.kB) % S.nB, P.th0);
  S.pb1 = ring_point(S.B, (S.j + 1 + S.kB) % S.nB, P.th0);
}

// one merge step: writes the triangle, advances the state
__device__ __forceinline__ void band_step(const TriParams &P, BandState &S, unsigned char *dst) {
  bool advA = S.i < S.nA && (S.j == S.nB || S.an <= S.bn);
  if (advA) {
    put_rec(dst, S.pa, S.pa1, S.pb);
    S.i++;
    S.pa = S.pa1;
    if (S.i < S.nA) {
      S.pa1 = ring_point(S.A, (S.i + 1) % S.nA, P.th0);
      S.an = keyA(S, S.i + 1, P.th0);
    }
  } else {
    put_rec(dst, S.pa, S.pb1, S.pb);
    S.j++;
    S.pb = S.pb1;
    if (S.j < S.nB) {
      S.pb1 = ring_point(S.B, (S.j + 1 + S.kB) % S.nB, P.th0);
      S.bn = keyB(S, S.j + 1, P.th0);
    }
  }
}

struct HoleState {
  Ring C;
  int M, m;
  f3 bp, p, p1;
};

__device__ void hole_open(const TriParams &P, int64_t g, int m, HoleState &S) {
  int n = P.hole_node[g];
  int64_t g0 = P.node_hole0[n];
  int2 H = P.hole_hdr[hbase(P.csr_off, n) + (g - g0)];
  float4 on = P.node[n];
  // hole entries reuse the Ring walker through a LoopRec-like view
  S.C.le = nullptr;
  S.C.arcs = P.arc + abase(P.csr_off, n);
  S.C.vs = P.vert + vbase(P.csr_off, n);
  S.C.cnt = H.y;
  S.C.ox = on.x; S.C.oy = on.y; S.C.oz = on.z;
  S.M = P.hole_M[g];
  S.m = m;
  float4 bp = P.hole_bp[g];
  S.bp = F3(on.x + bp.x, on.y + bp.y, on.z + bp.z);
}

__device__ __forceinline__ f3 hole_point(const TriParams &P, const HoleEnt *he, const HoleState &S, int idx) {
  int e = 0;
  while (e + 1 < S.C.cnt && he[e + 1].cum <= idx) e++;
  uint32_t af = he[e].arc_fwd;
  const ArcRec A = S.C.arcs[af & 0xffff];
  int N = arc_N(A.dt, P.th0);
  int j = idx - he[e].cum;
  f3 p = arc_point(A, S.C.vs, N, (af >> 16) ? j : N - j);
  return F3(S.C.ox + p.x, S.C.oy + p.y, S.C.oz + p.z);
}

__global__ void __launch_bounds__(EMIT_T) k_emit(TriParams P, int64_t first, int64_t count, unsigned char *out) {
  extern __shared__ __align__(128) unsigned char stage[];
  const int64_t chunk0 = first + (int64_t)blockIdx.x * EMIT_TPC;
  int64_t chunk_n = count - (int64_t)blockIdx.x * EMIT_TPC;
  if (chunk_n > EMIT_TPC) chunk_n = EMIT_TPC;
  const int64_t t0 = chunk0 + (int64_t)threadIdx.x * EMIT_R;
  int64_t tend = chunk0 + chunk_n;
  int64_t t = t0;
  int64_t t1 = t0 + EMIT_R < tend ? t0 + EMIT_R : tend;
  while (t < t1) {
    if (t < P.n_tri_band) {
      int64_t s = upper_bound64(P.strut_off, 0, P.S + 1, t) - 1;
      int q = (int)(t - P.strut_off[s]);
      BandState S;
      band_open(P, s, q, S);
      int64_t bend = P.strut_off[s + 1];
      while (t < t1 && t < bend) {
        band_step(P, S, stage + (t - chunk0) * REC);
        t++;
      }
    } else {
      int64_t tl = t - P.n_tri_band;
      int64_t g = upper_bound64(P.hole_off, 0, P.H + 1, tl) - 1;
      int m = (int)(tl - P.hole_off[g]);
      HoleState S;
      hole_open(P, g, m, S);
      int n = P.hole_node[g];
      int2 H = P.hole_hdr[hbase(P.csr_off, n) + (g - P.node_hole0[n])];
      const HoleEnt *he = P.hole_ent + hebase(P.csr_off, n) + H.x;
      int64_t hend = P.n_tri_band + P.hole_off[g + 1];
      S.p = hole_point(P, he, S, S.m);
      while (t < t1 && t < hend) {
        S.p1 = hole_point(P, he, S, (S.m + 1) % S.M);
        put_rec(stage + (t - chunk0) * REC, S.bp, S.p, S.p1);
        S.p = S.p1;
        S.m++;
        t++;
      }
    }
  }
  // chunk -> global: TMA bulk store of the 16-byte-aligned body, plain stores for the tail
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int64_t bytes = chunk_n * REC;
  const int64_t body = bytes & ~(int64_t)15;
  unsigned char *gdst = out + (chunk0 - first) * REC;
  if (threadIdx.x == 0 && body > 0) {
    uint32_t saddr = (uint32_t)__cvta_generic_to_shared(stage);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(saddr), "r"((uint32_t)body)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  for (int64_t b = body + threadIdx.x; b < bytes; b += EMIT_T) gdst[b] = stage[b];
  if (threadIdx.x == 0 && body > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncthreads();
}

TriParams make_params(lmm_ctx *c) {
  TriParams P;
  P.node = (const float4 *)c->node.p;
  P.csr_off = (const int *)c->csr_off.p;
  P.ends = (const int2 *)c->ends.p;
  P.strut_csr = (const int2 *)c->strut_csr.p;
  P.node_hdr = (const int4 *)c->node_hdr.p;
  P.vert = (const float4 *)c->vert.p;
  P.arc = (const ArcRec *)c->arc.p;
  P.loop_hdr = (const int2 *)c->loop_hdr.p;
  P.loop = (LoopRec *)c->loop.p;
  P.hole_hdr = (const int2 *)c->hole_hdr.p;
  P.hole_ent = (HoleEnt *)c->hole_ent.p;
  P.th0 = c->th0;
  P.S = c->S;
  P.N = c->N;
  P.band = (int4 *)c->band.p;
  P.band_cnt = (int64_t *)c->tmp64.p;
  P.strut_off = (const int64_t *)c->strut_off.p;
  P.node_hole0 = (const int64_t *)c->node_hole0_64.p;
  P.hole_M = (int *)c->hole_M.p;
  P.hole_off = (const int64_t *)c->hole_off.p;
  P.hole_bp = (float4 *)c->hole_bp.p;
  P.hole_node = (int *)c->hole_node.p;
  P.H = c->H;
  P.n_tri_band = c->n_tri_band;
  return P;
}

}  // namespace

int triangulate_count(lmm_ctx *c) {
  const int64_t S = c->S, N = c->N;
  int rc;
  if ((rc = dev_alloc(c->band, sizeof(int4) * (S + 1)))) return rc;
  if ((rc = dev_alloc(c->strut_off, sizeof(int64_t) * (S + 1)))) return rc;
  if ((rc = dev_alloc(c->tmp64, sizeof(int64_t) * ((S > N ? S : N) + 2)))) return rc;
  if ((rc = dev_alloc(c->node_hole0, sizeof(int) * (N + 1)))) return rc;
  if ((rc = dev_alloc(c->node_hole0_64, sizeof(int64_t) * (N + 1)))) return rc;
  const int T = 256;
  TriParams P = make_params(c);
  {
    KTimer t(c, LMM_K_COUNT);
    if (S) (c->n_launch++), k_band_count<<<(unsigned)((S + T - 1) / T), T, 0, c->stream>>>(P);
    if (N) (c->n_launch++), k_node_nholes<<<(unsigned)((N + T - 1) / T), T, 0, c->stream>>>((const int4 *)c->node_hdr.p, N, (int *)c->node_hole0.p);
    CUDA_TRY(cudaGetLastError());
  }
  if ((rc = scan_exclusive_i64(c, (const int64_t *)c->tmp64.p, (int64_t *)c->strut_off.p, S, &c->n_tri_band))) return rc;
  if ((rc = scan_exclusive_i32_to_i64(c, (const int *)c->node_hole0.p, (int64_t *)c->node_hole0_64.p, N, &c->H))) return rc;
  const int64_t H = c->H;
  if ((rc = dev_alloc(c->hole_M, sizeof(int) * (H + 1)))) return rc;
  if ((rc = dev_alloc(c->hole_off, sizeof(int64_t) * (H + 1)))) return rc;
  if ((rc = dev_alloc(c->hole_bp, sizeof(float4) * (H + 1)))) return rc;
  if ((rc = dev_alloc(c->hole_node, sizeof(int) * (H + 1)))) return rc;
  P = make_params(c);
  {
    KTimer t(c, LMM_K_COUNT);
    if (N) (c->n_launch++), k_hole_count<<<(unsigned)((N + T - 1) / T), T, 0, c->stream>>>(P);
    CUDA_TRY(cudaGetLastError());
  }
  int64_t hole_tri = 0;
  if ((rc = scan_exclusive_i32_to_i64(c, (const int *)c->hole_M.p, (int64_t *)c->hole_off.p, H, &hole_tri))) return rc;
  c->n_tri = c->n_tri_band + hole_tri;
  return LMM_OK;
}

int triangulate_emit(lmm_ctx *c, int64_t first, int64_t count, void *out_dev, cudaStream_t st) {
  if (count <= 0) return LMM_OK;
  TriParams P = make_params(c);
  const size_t smem = (size_t)EMIT_TPC * REC;
  static bool attr_set = false;
  if (!attr_set) {
    CUDA_TRY(cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  int64_t grid = (count + EMIT_TPC - 1) / EMIT_TPC;
  KTimer t(c, LMM_K_EMIT);
  (c->n_launch++), k_emit<<<(unsigned)grid, EMIT_T, smem, st>>>(P, first, count, (unsigned char *)out_dev);
  CUDA_TRY(cudaGetLastError());
  return LMM_OK;
}
