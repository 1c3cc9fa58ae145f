// triangulate.cu -- resolution-parametric triangulation of the meta-mesh
// (Sec. 5: Eq. 11 subdivision counts, Eq. 12 uniform parameters, strut bands
// "by connecting these vertices", Eq. 13 hole fans, Algorithm 1).
//
// Count pass (one thread per strut / per node): N per arc from the chord error, loop
// point counts, the band rotation, hole sizes and fan centres; device scans give the
// output offsets; then every band's stitch merge is run once and stored as one bit per
// triangle (advance ring A / ring B) with a per-32-triangle prefix count, and a map from
// output chunk to its first band/hole.
//
// Emit pass: output-centric persistent CTAs, each owning 1024-triangle chunks of the
// global order.  A thread takes 4 consecutive triangles: its ring positions come from
// the merge bits in O(1), it walks both rings with incremental cursors and computes one
// new Eq. 12 point per triangle.  The 50-byte STL records are assembled in shared
// memory and leave with one TMA bulk store (cp.async.bulk.global.shared::cta) per chunk.
//
// Decision arithmetic (N, stitch keys, band rotation, merge) is binary32 with the
// operation order of DESIGN.md Sec. 4.5 written with explicit round-to-nearest
// intrinsics (never contracted); geometry uses the fast paths.
#include "lmm_internal.h"

namespace {

constexpr int TPC = 1024;       // triangles per emit chunk (51 200 B of records)
constexpr int EMIT_T = 256;     // threads per emit CTA
constexpr int EMIT_R = TPC / EMIT_T;
constexpr int REC = 50;
constexpr int MAXSB = 64;       // band offsets cached per chunk

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
  int64_t n_tri_band, n_tri;
  uint32_t *mbits;          // merge bits, bit t = triangle t advances ring A
  int *macc;                // [word] A-advances of the band before the word's first bit
  int *cmap;                // [chunk] first band (band region) / hole (hole region)
  int64_t n_chunks;
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

// LoopRec.arc_fwd = arc | fwd << 16 | N << 17 (N written by the count pass)
__device__ __forceinline__ int le_arc(uint32_t af) { return af & 0xffff; }
__device__ __forceinline__ int le_fwd(uint32_t af) { return (af >> 16) & 1; }
__device__ __forceinline__ int le_N(uint32_t af) { return af >> 17; }

// Eq. 12 point jj of an arc, node-local; the endpoints are the shared vertices exactly
__device__ __forceinline__ f3 arc_point(const ArcRec &A, const float4 *vslab, int N, int jj) {
  if (jj == 0 || jj == N) {
    int v = jj == 0 ? (A.ids >> 16) & 0xff : (A.ids >> 24);
    float4 p = __ldg(&vslab[v]);
    return F3(p.x, p.y, p.z);
  }
  float t = A.t0 + (float)jj * (A.dt / (float)N);
  t = t - LMM_TWO_PI_F * rintf(t * (1.0f / LMM_TWO_PI_F));
  float s, c;
  __sincosf(t, &s, &c);
  return F3(fmaf(A.ax, s, fmaf(A.bx, c, A.ox)), fmaf(A.ay, s, fmaf(A.by, c, A.oy)), fmaf(A.az, s, fmaf(A.bz, c, A.oz)));
}

__device__ __forceinline__ ArcRec load_arc(const ArcRec *p) {
  const float4 *q = reinterpret_cast<const float4 *>(p);
  float4 x = __ldg(q), y = __ldg(q + 1), z = __ldg(q + 2);
  ArcRec a;
  a.ids = __float_as_uint(x.x); a.t0 = x.y; a.dt = x.z; a.ox = x.w;
  a.oy = y.x; a.oz = y.y; a.ax = y.z; a.ay = y.w;
  a.az = z.x; a.bx = z.y; a.by = z.z; a.bz = z.w;
  return a;
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
      uint32_t af = la[i].arc_fwd & 0x1ffffu;
      int N = arc_N(aa[le_arc(af)].dt, P.th0);
      la[i].arc_fwd = af | ((uint32_t)N << 17);
      la[i].cum = nA;
      nA += N;
    }
    for (int i = 0; i < LB.y; i++) {
      uint32_t af = lb[i].arc_fwd & 0x1ffffu;
      int N = arc_N(ab[le_arc(af)].dt, P.th0);
      lb[i].arc_fwd = af | ((uint32_t)N << 17);
      lb[i].cum = nB;
      nB += N;
    }
    if (nA > 0 && nB > 0) {
      // rotation of ring B: first point minimising its angle relative to A's start
      float a0 = la[0].phs;
      float best = 0.0f;
      int idx = 0;
      for (int i = 0; i < LB.y; i++) {
        float phs = lb[i].phs, dph = lb[i].dph;
        int N = le_N(lb[i].arc_fwd);
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

// sequential cursor over a ring's stitch keys (point index increases; wraps once)
struct KeyCursor {
  const LoopRec *le;
  int cnt, e, cum, N;
  float phs, dph;
  __device__ void load(int ee) {
    e = ee;
    LoopRec L = le[e];
    cum = L.cum; N = le_N(L.arc_fwd); phs = L.phs; dph = L.dph;
  }
  __device__ float key(int idx) {
    if (idx < cum) load(0);
    while (idx >= cum + N && e + 1 < cnt) load(e + 1);
    return key_at(phs, dph, N, idx - cum);
  }
};

// the stitch merge of every band, once: bit t = 1 iff triangle t advances ring A
__global__ void k_band_merge(TriParams P) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= P.S) return;
  int4 bd = P.band[s];
  const int nA = bd.x, nB = bd.y, kB = bd.z;
  if (nA + nB == 0) return;
  int2 e = P.ends[s];
  int2 ce = P.strut_csr[s];
  int2 LA = P.loop_hdr[ce.x], LB = P.loop_hdr[ce.y];
  KeyCursor A, B;
  A.le = P.loop + lbase(P.csr_off, e.x) + LA.x; A.cnt = LA.y; A.load(0);
  B.le = P.loop + lbase(P.csr_off, e.y) + LB.x; B.cnt = LB.y; B.load(0);
  const float a0 = A.phs;
  const float b0 = wrap_rel(B.key(kB), a0);
  const int64_t base = P.strut_off[s];
  const int64_t end = base + nA + nB;
  int i = 0, j = 0;
  float an = (1 < nA) ? __fsub_rn(A.key(1), a0) : LMM_TWO_PI_F;
  float bn = (1 < nB) ? wrap_rel(B.key((1 + kB) % nB), a0) : __fadd_rn(b0, LMM_TWO_PI_F);
  uint32_t word = 0;
  for (int64_t t = base; t < end; t++) {
    if ((t & 31) == 0) P.macc[t >> 5] = i;
    bool advA = i < nA && (j == nB || an <= bn);
    if (advA) {
      word |= 1u << (t & 31);
      i++;
      if (i < nA) an = (i + 1 < nA) ? __fsub_rn(A.key(i + 1), a0) : LMM_TWO_PI_F;
    } else {
      j++;
      if (j < nB) bn = (j + 1 < nB) ? wrap_rel(B.key((j + 1 + kB) % nB), a0) : __fadd_rn(b0, LMM_TWO_PI_F);
    }
    if ((t & 31) == 31 || t + 1 == end) {
      int64_t w = t >> 5;
      bool full = (w << 5) >= base && (w << 5) + 31 < end;
      if (full) P.mbits[w] = word;
      else if (word) atomicOr(&P.mbits[w], word);
      word = 0;
    }
  }
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
      uint32_t af = he[H.x + i].arc_fwd & 0x1ffffu;
      int N = arc_N(as[le_arc(af)].dt, P.th0);
      he[H.x + i].arc_fwd = af | ((uint32_t)N << 17);
      he[H.x + i].cum = M;
      M += N;
    }
    // Eq. 13 fan centre: barycentre of the contour vertices, direction regularised by
    // the contour's outward (Newell) normal (reading R7)
    float bx = 0.f, by = 0.f, bz = 0.f, nx = 0.f, ny = 0.f, nz = 0.f;
    f3 first = F3(0.f, 0.f, 0.f), prev = first;
    bool have = false;
    for (int i = 0; i < H.y; i++) {
      uint32_t af = he[H.x + i].arc_fwd;
      const ArcRec A = as[le_arc(af)];
      int fwd = le_fwd(af);
      int N = le_N(af);
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

// chunk -> first band containing the chunk's first triangle
__global__ void k_chunk_map_bands(TriParams P) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= P.S) return;
  int64_t b = P.strut_off[s], e = P.strut_off[s + 1];
  if (b == e) return;
  for (int64_t c = (b + TPC - 1) / TPC; c * TPC < e; c++) P.cmap[c] = (int)s;
}
__global__ void k_chunk_map_holes(TriParams P) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= P.H) return;
  int64_t b = P.n_tri_band + P.hole_off[g], e = P.n_tri_band + P.hole_off[g + 1];
  if (b == e) return;
  for (int64_t c = (b + TPC - 1) / TPC; c * TPC < e; c++) P.cmap[c] = (int)g;
}

// ---------------------------------------------------------------------------------
// emit pass
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void put_rec(unsigned char *dst, f3 a, f3 b, f3 c) {
  f3 u = f_sub(b, a), v = f_sub(c, a);
  float nx = u.y * v.z - u.z * v.y, ny = u.z * v.x - u.x * v.z, nz = u.x * v.y - u.y * v.x;
  float l2 = nx * nx + ny * ny + nz * nz;
  float il = l2 > 0.0f ? rsqrtf(l2) : 0.0f;
  float f[12] = {nx * il, ny * il, nz * il, a.x, a.y, a.z, b.x, b.y, b.z, c.x, c.y, c.z};
  if ((((uintptr_t)dst) & 3) == 0) {
    uint32_t *d32 = reinterpret_cast<uint32_t *>(dst);
#pragma unroll
    for (int i = 0; i < 12; i++) d32[i] = __float_as_uint(f[i]);
    reinterpret_cast<uint16_t *>(dst)[24] = 0;
  } else {
    uint16_t *d16 = reinterpret_cast<uint16_t *>(dst);   // records are 2-byte aligned
    d16[0] = (uint16_t)(__float_as_uint(f[0]) & 0xffffu);
    uint32_t *d32 = reinterpret_cast<uint32_t *>(dst + 2);
#pragma unroll
    for (int i = 0; i < 11; i++) d32[i] = __funnelshift_r(__float_as_uint(f[i]), __float_as_uint(f[i + 1]), 16);
    d32[11] = __float_as_uint(f[11]) >> 16;   // high half of f11 + attribute 0
  }
}

// point cursor over a ring (node-local arcs -> absolute positions)
struct PtCursor {
  const LoopRec *le;
  const ArcRec *arcs;
  const float4 *vs;
  int cnt, e, cum, N, fwd;
  ArcRec A;
  float ox, oy, oz;
  __device__ void load(int ee) {
    e = ee;
    LoopRec L = le[e];
    cum = L.cum; N = le_N(L.arc_fwd); fwd = le_fwd(L.arc_fwd);
    A = load_arc(arcs + le_arc(L.arc_fwd));
  }
  __device__ f3 point(int idx) {
    if (idx < cum) load(0);
    while (idx >= cum + N && e + 1 < cnt) load(e + 1);
    int j = idx - cum;
    f3 p = arc_point(A, vs, N, fwd ? j : N - j);
    return F3(ox + p.x, oy + p.y, oz + p.z);
  }
};

// A-advances of band [base, ...) before triangle t
__device__ __forceinline__ int merge_rank(const TriParams &P, int64_t base, int64_t t) {
  int64_t w = t >> 5;
  uint32_t word = __ldg(&P.mbits[w]);
  int sh = (int)(t - (w << 5));
  uint32_t below = sh ? (word & ((1u << sh) - 1u)) : 0u;
  if (base > (w << 5)) {
    int bs = (int)(base - (w << 5));
    return __popc(below & ~((1u << bs) - 1u));
  }
  return __ldg(&P.macc[w]) + __popc(below);
}

__device__ void emit_band_run(const TriParams &P, int64_t s, int64_t t, int64_t t1, unsigned char *stage, int64_t sbase) {
  const int2 e = P.ends[s];
  const int2 ce = P.strut_csr[s];
  const int4 bd = P.band[s];
  const int nA = bd.x, nB = bd.y, kB = bd.z;
  const int64_t base = P.strut_off[s];
  const int2 LA = P.loop_hdr[ce.x], LB = P.loop_hdr[ce.y];
  const float4 oa = P.node[e.x], ob = P.node[e.y];
  PtCursor A, B;
  A.le = P.loop + lbase(P.csr_off, e.x) + LA.x; A.arcs = P.arc + abase(P.csr_off, e.x);
  A.vs = P.vert + vbase(P.csr_off, e.x); A.cnt = LA.y; A.ox = oa.x; A.oy = oa.y; A.oz = oa.z;
  B.le = P.loop + lbase(P.csr_off, e.y) + LB.x; B.arcs = P.arc + abase(P.csr_off, e.y);
  B.vs = P.vert + vbase(P.csr_off, e.y); B.cnt = LB.y; B.ox = ob.x; B.oy = ob.y; B.oz = ob.z;
  A.load(0);
  B.load(0);
  int i = merge_rank(P, base, t);
  int j = (int)(t - base) - i;
  f3 pa = A.point(i % nA);
  int jb = (j + kB) % nB;
  f3 pb = B.point(jb);
  for (; t < t1; t++) {
    bool advA = (__ldg(&P.mbits[t >> 5]) >> (t & 31)) & 1u;
    unsigned char *dst = stage + (t - sbase) * REC;
    if (advA) {
      i++;
      f3 pa1 = A.point(i == nA ? 0 : i);
      put_rec(dst, pa, pa1, pb);
      pa = pa1;
    } else {
      j++;
      int jb1 = jb + 1 == nB ? 0 : jb + 1;
      f3 pb1 = B.point(jb1);
      put_rec(dst, pa, pb1, pb);
      pb = pb1;
      jb = jb1;
    }
  }
}

__device__ void emit_hole_run(const TriParams &P, int64_t g, int64_t t, int64_t t1, unsigned char *stage, int64_t sbase) {
  const int n = P.hole_node[g];
  const int64_t g0 = P.node_hole0[n];
  const int2 H = P.hole_hdr[hbase(P.csr_off, n) + (g - g0)];
  const float4 on = P.node[n];
  const float4 bp4 = P.hole_bp[g];
  const f3 bp = F3(on.x + bp4.x, on.y + bp4.y, on.z + bp4.z);
  const int M = P.hole_M[g];
  const int64_t hb = P.n_tri_band + P.hole_off[g];
  // hole entries have the loop-entry layout's first two words (arc_fwd, cum)
  const HoleEnt *he = P.hole_ent + hebase(P.csr_off, n) + H.x;
  const ArcRec *arcs = P.arc + abase(P.csr_off, n);
  const float4 *vs = P.vert + vbase(P.csr_off, n);
  int m = (int)(t - hb);
  int e = 0;
  auto point = [&](int idx) -> f3 {
    if (idx < he[e].cum) e = 0;
    while (e + 1 < H.y && idx >= he[e + 1].cum) e++;
    uint32_t af = he[e].arc_fwd;
    ArcRec A = load_arc(arcs + le_arc(af));
    int N = le_N(af), j = idx - he[e].cum;
    f3 p = arc_point(A, vs, N, le_fwd(af) ? j : N - j);
    return F3(on.x + p.x, on.y + p.y, on.z + p.z);
  };
  f3 p = point(m);
  for (; t < t1; t++) {
    m++;
    f3 p1 = point(m == M ? 0 : m);
    put_rec(stage + (t - sbase) * REC, bp, p, p1);
    p = p1;
  }
}

__device__ __forceinline__ int64_t upper_bound64(const int64_t *a, int64_t lo, int64_t hi, int64_t x) {
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (__ldg(&a[m]) <= x) lo = m + 1; else hi = m;
  }
  return lo;
}

__global__ void __launch_bounds__(EMIT_T) k_emit(TriParams P, int64_t first, int64_t count, unsigned char *out) {
  extern __shared__ __align__(128) unsigned char stage[];
  __shared__ int64_t soff[MAXSB + 1];
  __shared__ int sb0, nsb;
  const int64_t last = first + count;
  const int64_t c0 = first / TPC, c1 = (last + TPC - 1) / TPC;
  const bool congruent = ((first % 8) == 0);   // record offsets then stay 16-byte congruent
  for (int64_t c = c0 + blockIdx.x; c < c1; c += gridDim.x) {
    const int64_t cs = c * TPC;
    const int64_t lo = cs > first ? cs : first;
    const int64_t hi = cs + TPC < last ? cs + TPC : last;
    // band offsets of this chunk into shared memory
    if (threadIdx.x == 0) {
      int b0 = lo < P.n_tri_band ? P.cmap[c] : -1;
      sb0 = b0;
      int cnt = 0;
      if (b0 >= 0) {
        int64_t lim = P.S - b0;
        cnt = (int)(lim < MAXSB ? lim : MAXSB);
      }
      nsb = cnt;
    }
    __syncthreads();
    if (sb0 >= 0)
      for (int k = threadIdx.x; k <= nsb; k += EMIT_T) soff[k] = P.strut_off[sb0 + k];
    __syncthreads();
    int64_t t = lo + (int64_t)threadIdx.x * EMIT_R;
    const int64_t tend = t + EMIT_R < hi ? t + EMIT_R : hi;
    while (t < tend) {
      if (t < P.n_tri_band) {
        int64_t s;
        if (sb0 >= 0 && t < soff[nsb]) {
          int a = 0, b = nsb;   // last k with soff[k] <= t
          while (b - a > 1) { int m = (a + b) >> 1; if (soff[m] <= t) a = m; else b = m; }
          s = sb0 + a;
        } else {
          s = upper_bound64(P.strut_off, 0, P.S + 1, t) - 1;
        }
        int64_t bend = P.strut_off[s + 1];
        int64_t t1 = tend < bend ? tend : bend;
        emit_band_run(P, s, t, t1, stage, cs);
        t = t1;
      } else {
        int64_t tl = t - P.n_tri_band;
        int64_t g = cs >= P.n_tri_band ? P.cmap[c] : 0;   // hole holding the chunk's first triangle
        g = upper_bound64(P.hole_off, g, P.H + 1, tl) - 1;
        int64_t hend = P.n_tri_band + P.hole_off[g + 1];
        int64_t t1 = tend < hend ? tend : hend;
        emit_hole_run(P, g, t, t1, stage, cs);
        t = t1;
      }
    }
    // chunk -> global: TMA bulk store of the 16-byte-aligned body, plain stores around it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int64_t sb = (lo - cs) * REC, se = (hi - cs) * REC;   // staging byte range
    unsigned char *gdst = out + (lo - first) * REC - sb;          // gdst[sb..se) <- stage[sb..se)
    int64_t bb = sb, be = sb;
    if (congruent) {
      bb = (sb + 15) & ~(int64_t)15;
      be = se & ~(int64_t)15;
      if (be < bb) be = bb;
    }
    if (threadIdx.x == 0 && be > bb) {
      uint32_t saddr = (uint32_t)__cvta_generic_to_shared(stage + bb);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst + bb), "r"(saddr),
                   "r"((uint32_t)(be - bb))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    for (int64_t b = sb + threadIdx.x; b < bb; b += EMIT_T) gdst[b] = stage[b];
    for (int64_t b = (be > bb ? be : bb) + threadIdx.x; b < se; b += EMIT_T) gdst[b] = stage[b];
    if (threadIdx.x == 0 && be > bb) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
  }
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
  P.n_tri = c->n_tri;
  P.mbits = (uint32_t *)c->mbits.p;
  P.macc = (int *)c->macc.p;
  P.cmap = (int *)c->cmap.p;
  P.n_chunks = (c->n_tri + TPC - 1) / TPC;
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
  const int64_t nwords = c->n_tri_band / 32 + 2;
  if ((rc = dev_alloc(c->mbits, sizeof(uint32_t) * nwords))) return rc;
  if ((rc = dev_alloc(c->macc, sizeof(int) * nwords))) return rc;
  P = make_params(c);
  {
    KTimer t(c, LMM_K_COUNT);
    CUDA_TRY(cudaMemsetAsync(c->mbits.p, 0, sizeof(uint32_t) * nwords, c->stream));
    if (N) (c->n_launch++), k_hole_count<<<(unsigned)((N + T - 1) / T), T, 0, c->stream>>>(P);
    if (S) (c->n_launch++), k_band_merge<<<(unsigned)((S + T - 1) / T), T, 0, c->stream>>>(P);
    CUDA_TRY(cudaGetLastError());
  }
  int64_t hole_tri = 0;
  if ((rc = scan_exclusive_i32_to_i64(c, (const int *)c->hole_M.p, (int64_t *)c->hole_off.p, H, &hole_tri))) return rc;
  c->n_tri = c->n_tri_band + hole_tri;
  const int64_t nch = (c->n_tri + TPC - 1) / TPC + 1;
  if ((rc = dev_alloc(c->cmap, sizeof(int) * nch))) return rc;
  P = make_params(c);
  {
    KTimer t(c, LMM_K_COUNT);
    if (S) (c->n_launch++), k_chunk_map_bands<<<(unsigned)((S + T - 1) / T), T, 0, c->stream>>>(P);
    if (H) (c->n_launch++), k_chunk_map_holes<<<(unsigned)((H + T - 1) / T), T, 0, c->stream>>>(P);
    CUDA_TRY(cudaGetLastError());
  }
  return LMM_OK;
}

int triangulate_emit(lmm_ctx *c, int64_t first, int64_t count, void *out_dev, cudaStream_t st) {
  if (count <= 0) return LMM_OK;
  TriParams P = make_params(c);
  const size_t smem = (size_t)TPC * REC;
  static bool attr_set = false;
  static int occ = 1;
  if (!attr_set) {
    CUDA_TRY(cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit, EMIT_T, smem));
    if (occ < 1) occ = 1;
    attr_set = true;
  }
  int64_t nch = (first + count + TPC - 1) / TPC - first / TPC;
  int64_t grid = (int64_t)c->n_sm * occ;
  if (grid > nch) grid = nch;
  KTimer t(c, LMM_K_EMIT);
  (c->n_launch++), k_emit<<<(unsigned)grid, EMIT_T, smem, st>>>(P, first, count, (unsigned char *)out_dev);
  CUDA_TRY(cudaGetLastError());
  return LMM_OK;
}
