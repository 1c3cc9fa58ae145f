// triangulate.cu -- resolution-parametric triangulation of the meta-mesh
// (Sec. 5: Eq. 11 subdivision counts, Eq. 12 uniform parameters, strut bands
// "by connecting these vertices", Eq. 13 hole fans, Algorithm 1).
//
// Count pass: Eq. 11 N per arc and the point offsets of every ring (one thread per strut
// end, a node's rings on consecutive threads), band sizes per strut, hole sizes and fan
// centres per node; device scans give the output offsets; then every band's rotation and
// stitch merge is run once (one thread per strut, forward key cursors) and stored as one bit
// per triangle (advance ring A / ring B) with a per-32-triangle prefix count, together with
// the band's 64-byte emit record; a map from 1024-triangle output chunks to their first
// band/hole bounds any requested range.
//
// Emit pass: warps grid-stride over the bands (then the hole fans) of the requested range.
// A band is fetched as its record, then its loop entries, arcs and start vertices (cp.async
// stages overlapped with the previous band); its ring points are computed once into a
// shared-memory cache sized per triangulation; lanes assemble pairs of 50-byte STL records
// (ring positions from ballot prefix-popcounts of the merge bits) in a per-warp staging
// buffer, which leaves as one TMA bulk copy (cp.async.bulk.global.shared::cta) per
// 56-triangle group on the 16-byte output grid.
//
// Decision arithmetic (N, stitch keys, band rotation, merge) is binary32 with the
// operation order of DESIGN.md Sec. 4.5 written with explicit round-to-nearest
// intrinsics (never contracted); geometry uses the fast paths.
#include "lmm_internal.h"

namespace {

constexpr int TPC = 1024;       // triangles per emit chunk (51 200 B of records)
constexpr int EMIT_T = 128;     // threads per emit CTA
constexpr int REC = 50;

// Everything the emit pass needs to start a band, written once per strut by k_band_merge
// (after the offsets scan), so that a band is fetched as one 64-byte record + its offset.
struct __align__(16) BandRec {
  int nA, nB, kB, lAc;   // ring sizes, ring-B rotation; lAc = first loop entry of ring A in
  int lBc;               //   its node's loop slab | entry count << 16 (lBc: ring B)
  unsigned aA, aB;       // arc slab base of each end node (3 off + 2 n; loop slab = 2 a)
  unsigned pA, pB;       // off + n of each end node (vertex slab = 2 p)
  float oax, oay, oaz, obx, oby, obz, pad;   // node centres
};
static_assert(sizeof(BandRec) == 64, "band record is 4 x 16 bytes");

struct TriParams {
  const float4 *node;
  const int *csr_off;
  const int2 *skey;         // [N] slab key of each node
  const int2 *csr_ent;
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
  BandRec *brec;            // [S] emit records
  const uint8_t *node_mask; // [N] or null
  const uint8_t *strut_mask;// [S] or null
  int64_t n_chunks;
};

__device__ __forceinline__ int arc_N(float dt, float th0) { return (int)floorf(__fdiv_rn(dt, th0)) + 1; }


__device__ __forceinline__ float wrap_rel(float b, float a0) {
  float r = __fsub_rn(b, a0);
  if (r < 0.0f) r = __fadd_rn(r, LMM_TWO_PI_F);
  if (r >= LMM_TWO_PI_F) r = __fsub_rn(r, LMM_TWO_PI_F);
  return r;
}

// slab bases of a node from its slab key (off, n) (spilled nodes: virtual keys)
__device__ __forceinline__ int64_t vbase(int2 k) { return slab_base(k.x, k.y, SLAB_V_K, SLAB_V_K0); }
__device__ __forceinline__ int64_t abase(int2 k) { return slab_base(k.x, k.y, SLAB_A_K, SLAB_A_K0); }
__device__ __forceinline__ int64_t lbase(int2 k) { return slab_base(k.x, k.y, SLAB_L_K, SLAB_L_K0); }
__device__ __forceinline__ int64_t hbase(int2 k) { return slab_base(k.x, k.y, SLAB_H_K, SLAB_H_K0); }
__device__ __forceinline__ int64_t hebase(int2 k) { return slab_base(k.x, k.y, SLAB_HE_K, SLAB_HE_K0); }

// LoopRec.arc_fwd = arc | fwd << 16 | N << 17 (N written by the count pass)
__device__ __forceinline__ int le_arc(uint32_t af) { return af & 0xffff; }
__device__ __forceinline__ int le_fwd(uint32_t af) { return (af >> 16) & 1; }
__device__ __forceinline__ int le_N(uint32_t af) { return af >> 17; }

// Eq. 12 point jj of an arc, node-local; the endpoints are the shared vertices exactly
__device__ __forceinline__ f3 arc_point(const ArcRec &A, const float4 *vslab, int N, int jj) {
  if (jj == 0 || jj == N) {
    int v = jj == 0 ? arc_vs(A.ids) : arc_ve(A.ids);
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
// Eq. 11 N of every arc of one ring and the running point offsets; returns the ring's
// point count.  Loads are issued four entries at a time ahead of the dependent stores.
__device__ __forceinline__ int ring_counts(LoopRec *__restrict__ le, int cnt, const ArcRec *__restrict__ arc, float th0) {
  int n = 0;
  for (int i0 = 0; i0 < cnt; i0 += 4) {
    uint32_t af[4];
    float dt[4];
    int vt[4];
#pragma unroll
    for (int k = 0; k < 4; k++) af[k] = i0 + k < cnt ? (le[i0 + k].arc_fwd & 0x1ffffu) : 0u;
#pragma unroll
    for (int k = 0; k < 4; k++) vt[k] = i0 + k < cnt ? (le[i0 + k].cum & LE_VID_MASK) : 0;
#pragma unroll
    for (int k = 0; k < 4; k++) dt[k] = i0 + k < cnt ? __ldg(&arc[le_arc(af[k])].dt) : 0.0f;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (i0 + k < cnt) {
        int N = arc_N(dt[k], th0);
        le[i0 + k].arc_fwd = af[k] | ((uint32_t)N << 17);
        le[i0 + k].cum = vt[k] | n;   // the start vertex stays in the top byte
        n += N;
      }
    }
  }
  return n;
}

// Eq. 11 counts of one ring (strut end) per thread.  Thread = CSR entry, so consecutive
// threads work on the same node's loop and arc slabs (coalesced, cache-friendly reads).
__global__ void k_ring_count(TriParams P, int64_t S2, int *ring_n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= S2) return;
  const int2 ent = P.csr_ent[i];
  const int2 e = P.ends[ent.x];
  const int n = ((unsigned)ent.y >> 31) ? e.y : e.x;   // the node this entry belongs to
  int nr = 0;
  if ((P.node_hdr[n].x & 0xff) == 0) {
    const int2 key = P.skey[n];
    const int2 L = P.loop_hdr[i];
    nr = ring_counts(P.loop + lbase(key) + L.x, L.y, P.arc + abase(key), P.th0);
  }
  ring_n[i] = nr;
}

// band sizes from the two rings of each strut (0 when masked out or an end node failed)
__global__ void k_band_count(TriParams P, const int *ring_n) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= P.S) return;
  int nA = 0, nB = 0;
  if (!P.strut_mask || P.strut_mask[s]) {
    const int2 ce = P.strut_csr[s];
    nA = ring_n[ce.x];
    nB = ring_n[ce.y];
    if (!(nA > 0 && nB > 0)) nA = nB = 0;   // the band rotation kB is found by k_band_merge
  }
  P.band[s] = make_int4(nA, nB, 0, 0);
  P.band_cnt[s] = (int64_t)nA + nB;
}

// Sequential cursor over a ring's stitch keys: key(idx) = phs_e + (idx - cum_e) * (dph_e / N_e)
// of the last entry e with cum_e <= idx; past the last entry's end the
// last entry is extrapolated.  Walked forward one point at a time (rem = points left in the
// current entry), re-seeked only where a ring wraps.
struct SeqKey {
  const LoopRec *le;
  int cnt, e, rem;
  float fj;      // index within the entry as a float (exact: < 2^24)
  float phs, step;
  __device__ void enter(int ee, int j0) {
    e = ee;
    const LoopRec L = le[e];
    const int N = le_N(L.arc_fwd);
    phs = L.phs;
    step = __fdiv_rn(L.dph, (float)N);   // same bits as dividing at every key
    fj = (float)j0;
    rem = N - j0;
  }
  __device__ void seek(int idx) {
    int ee = 0, cum = 0;
    for (;;) {
      const LoopRec L = le[ee];
      const int N = le_N(L.arc_fwd);
      cum = le_cum(L.cum);
      if (idx < cum + N || ee + 1 >= cnt) break;
      ee++;
    }
    enter(ee, idx - cum);
  }
  __device__ float key() const { return __fadd_rn(phs, __fmul_rn(fj, step)); }
  __device__ void next() {
    fj += 1.0f;
    if (--rem == 0 && e + 1 < cnt) enter(e + 1, 0);
  }
};

// the stitch merge of every band, once: bit t = 1 iff triangle t advances ring A
__global__ void k_band_merge(TriParams P) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= P.S) return;
  int4 bd = P.band[s];
  const int nA = bd.x, nB = bd.y;
  float4 *rq = reinterpret_cast<float4 *>(P.brec + s);
  if (nA + nB == 0) { rq[0] = make_float4(0.f, 0.f, 0.f, 0.f); return; }
  int2 e = P.ends[s];
  int2 ce = P.strut_csr[s];
  int2 LA = P.loop_hdr[ce.x], LB = P.loop_hdr[ce.y];
  {
    const int2 kA = P.skey[e.x], kB = P.skey[e.y];
    const float4 na = P.node[e.x], nb = P.node[e.y];
    rq[1] = make_float4(__int_as_float(LB.x | (LB.y << 16)), __uint_as_float(3u * kA.x + 2u * kA.y),
                        __uint_as_float(3u * kB.x + 2u * kB.y), __uint_as_float((unsigned)(kA.x + kA.y)));
    rq[2] = make_float4(__uint_as_float((unsigned)(kB.x + kB.y)), na.x, na.y, na.z);
    rq[3] = make_float4(nb.x, nb.y, nb.z, 0.0f);
  }
  SeqKey A, B;
  A.le = P.loop + lbase(P.skey[e.x]) + LA.x; A.cnt = LA.y;
  B.le = P.loop + lbase(P.skey[e.y]) + LB.x; B.cnt = LB.y;
  A.enter(0, 0);
  const float a0 = A.phs;     // ring A first entry phi
  // rotation of ring B: its first point with the smallest angle relative to A's start
  int kB = 0;
  float best = __int_as_float(0x7f800000);   // first index of the minimum (strict <)
  B.enter(0, 0);
  for (int j = 0; j < nB; j++, B.next()) {
    const float r = wrap_rel(B.key(), a0);
    if (r < best) { best = r; kB = j; }
  }
  P.band[s].z = kB;
  rq[0] = make_float4(__int_as_float(nA), __int_as_float(nB), __int_as_float(kB), __int_as_float(LA.x | (LA.y << 16)));
  const float b0 = best;   // = wrap_rel(key_B(kB), a0)
  // merge: an = key_A(i + 1) - a0 (2 pi after the last point), bn = wrap(key_B(kB + j + 1)) (b0 +
  // 2 pi after the last); triangle q advances ring A iff i < nA and (j == nB or an <= bn)
  const int64_t base = P.strut_off[s];
  const int n = nA + nB;
  const int sb = (int)(base & 31);
  uint32_t *mw = P.mbits + (base >> 5);
  int *ma = P.macc + (base >> 5);
  int i = 0, j = 0;
  int jb = 1 + kB >= nB ? 1 + kB - nB : 1 + kB;   // ring-B index of B's next point
  if (nA > 1) A.seek(1);
  if (nB > 1) B.seek(jb);
  float an = (1 < nA) ? __fsub_rn(A.key(), a0) : LMM_TWO_PI_F;
  float bn = (1 < nB) ? wrap_rel(B.key(), a0) : __fadd_rn(b0, LMM_TWO_PI_F);
  const int nw = (sb + n + 31) >> 5;
  for (int w = 0; w < nw; w++) {
    const int q0 = w == 0 ? 0 : 32 * w - sb;
    const int q1 = 32 * (w + 1) - sb < n ? 32 * (w + 1) - sb : n;
    if (w > 0) ma[w] = i;   // A-advances before the word's first bit
    // an / bn become +inf once their ring is exhausted, so "i < nA && (j == nB || an <= bn)"
    // is just "an <= bn" (both exhausted only after the last step)
    uint32_t word = 0, bit = 1u << ((sb + q0) & 31);
    for (int q = q0; q < q1; q++, bit <<= 1) {
      if (an <= bn) {
        word |= bit;
        i++;
        if (i + 1 < nA) { A.next(); an = __fsub_rn(A.key(), a0); }
        else an = i < nA ? LMM_TWO_PI_F : __int_as_float(0x7f800000);
      } else {
        j++;
        if (j + 1 < nB) {
          if (++jb == nB) { jb = 0; B.enter(0, 0); } else B.next();
          bn = wrap_rel(B.key(), a0);
        } else bn = j < nB ? __fadd_rn(b0, LMM_TWO_PI_F) : __int_as_float(0x7f800000);
      }
    }
    // a word is the band's alone when it starts at or after the band start and ends inside it
    const bool own = 32 * w >= sb && 32 * w + 31 <= sb + n - 1;
    if (own) mw[w] = word;
    else if (word) atomicOr(&mw[w], word);
  }
  if (sb == 0) ma[0] = 0;
}

__global__ void k_node_nholes(const int4 *hdr, int64_t N, const uint8_t *mask, int *nh) {
  int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= N) return;
  int4 h = hdr[n];
  nh[n] = ((h.x & 0xff) == 0 && (!mask || mask[n])) ? (h.z & 0xffff) : 0;
}

__global__ void k_hole_count(TriParams P) {
  int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= P.N) return;
  int64_t g0 = P.node_hole0[n], g1 = P.node_hole0[n + 1];
  if (g0 == g1) return;
  const float4 on = P.node[n];
  const float R = on.w;
  const int2 key = P.skey[n];
  const float4 *vs = P.vert + vbase(key);
  const ArcRec *as = P.arc + abase(key);
  const int2 *hh = P.hole_hdr + hbase(key);
  HoleEnt *he = P.hole_ent + hebase(key);
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
    // sums taken relative to the first contour point p0 (the Newell sum is translation
    // invariant for a closed contour; this keeps small holes well conditioned in binary32)
    float bx = 0.f, by = 0.f, bz = 0.f, nx = 0.f, ny = 0.f, nz = 0.f;
    f3 p0 = F3(0.f, 0.f, 0.f), prev = p0;
    bool have = false;
    for (int i = 0; i < H.y; i++) {
      uint32_t af = he[H.x + i].arc_fwd;
      const ArcRec A = as[le_arc(af)];
      int fwd = le_fwd(af);
      int N = le_N(af);
      for (int j = 0; j < N; j++) {
        f3 p = arc_point(A, vs, N, fwd ? j : N - j);
        if (!have) { p0 = p; have = true; prev = F3(0.f, 0.f, 0.f); continue; }
        f3 q = f_sub(p, p0);
        bx += q.x; by += q.y; bz += q.z;
        f3 cr = f_cross(prev, q);
        nx += cr.x; ny += cr.y; nz += cr.z;
        prev = q;
      }
    }
    float inv = 1.0f / (float)M;
    const float n2 = nx * nx + ny * ny + nz * nz;
    float nl = n2 > 0.0f ? rsqrtf(n2) : 0.0f;   // a contour without area keeps Eq. 13's b - o
    float dx = (p0.x + bx * inv) + R * nx * nl, dy = (p0.y + by * inv) + R * ny * nl, dz = (p0.z + bz * inv) + R * nz * nl;
    float dl = R * rsqrtf(dx * dx + dy * dy + dz * dz);
    // a contour of two points (a lune of two one-segment arcs: coincident chords) encloses no
    // area at this chord error and gets no fan (reading R7)
    P.hole_M[g] = M == 2 ? 0 : M;
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

// Warp-per-band emission.  Warps grid-stride over the strut bands (then the hole fans)
// that intersect [first, first+count).  A band's ring data -- both rings' loop entries and
// arc records -- sits in shared memory; every ring point is computed once, in parallel
// (the entry of a point comes from a ballot/redux count of the entry starts below it).
// Bands whose rings exceed the point cache (pcap points) are walked in windows of pcap - 2
// merge steps instead.
// Triangles then go in groups of 64 whose output offset is 16-byte aligned: lane l
// assembles records 2l and 2l+1 (100 bytes = 25 aligned words), its ring positions
// following from ballot prefix-popcounts of the merge bits; the group leaves the per-warp
// staging buffer as 16-byte vector stores.
//
// The next band's data is fetched with cp.async straight into shared memory in four
// dependent stages overlapped with the current band: header (before its points), loop
// headers / centres / offsets (after its points), loop entries (after its first group)
// and arc records (after its last group).  No registers are held across a band and no
// block-level barriers are used.
constexpr int EW = EMIT_T / 32;   // warps per CTA
#ifndef LMM_EMIT_BAND_MINB
#define LMM_EMIT_BAND_MINB 7   // k_emit CTAs per SM the registers are sized for (72 registers)
#endif
constexpr int PCAP_MIN = 152;     // ring points cached per band (both rings), runtime-sized
constexpr int PCAP_MAX = 640;     //   from the mean band size (triangulate_emit)
constexpr int GRP = 56;           // triangles per aligned group (2800 B; 28 lanes x 2 records)
constexpr int MAXRE = 32;         // ring entries per ring (>= MAXLOOP of the meta-mesh)
constexpr int MAXRA = 8;          // arc records (and entry start vertices) cached per ring

constexpr int GW = 64;            // triangles per group of the CTA-window path (32 lanes x 2 records)

// a loop entry of a span window as the point pass reads it (built in place from the raw arc
// record + start vertex that cp.async staged in the same slot)
struct __align__(16) PtEnt {
  float t0, dq;               // Eq. 12: t = t0 + jj * dq, dq = dt / N (fast division, as arc_pt)
  float ox, oy, oz, ax, ay, az, bx, by, bz;   // Eq. 1 arc frame (node-local)
  float cx, cy, cz;           // node centre of the ring
  int nf;                     // N | fwd << 16
  int P0;                     // cache position of the entry's point j = 0
  int wj;                     // points j >= wj sit `off` lower (ring-B rotation wraps inside the entry)
  int dupj;                   // point j == dupj is also stored at its position + off (ring closure copy)
  int off;                    // nA (ring A) / nB (ring B)
  int pad;                    // est: the entry's first point in the window's flattened point order
};
static_assert(sizeof(PtEnt) == 80, "window entry is 80 bytes");

// per-warp shared memory: fixed part, then the point cache (pcap x float2, pcap x float)
struct __align__(16) WarpRing {
  ArcRec arc[2][MAXRA];
  float4 vq[2][MAXRA];    // start vertex of each cached entry (node-local)
  LoopRec le[2][MAXRE];   // loop entries (arc | fwd | N, phs, dph, cum); holes: arc_fwd, cum
  uint4 stage[GRP * REC / 16];
};
__host__ __device__ constexpr int ring_bytes(int pcap) {
  return (int)((sizeof(WarpRing) + (size_t)pcap * 12 + 15) / 16 * 16);
}
// the point cache of one warp: xy pairs and z, capacity cap (cap - 2 merge steps per window)
struct Pts {
  float2 *xy;
  float *z;
  int cap;
};

template <int BYTES>
__device__ __forceinline__ void cp_async(void *sdst, const void *gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(sa), "l"(gsrc), "n"(BYTES) : "memory");
}
// all of this thread's cp.async done, then visible to the warp
__device__ __forceinline__ void cp_async_wait_warp() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncwarp();
}

// stage 1 of a band: its record (lanes 0-3) and triangle offset (lane 4)
__device__ __forceinline__ void fetch_rec(const TriParams &P, int s, BandRec &h, long long &base, int lane) {
  if (lane < 4) cp_async<16>(reinterpret_cast<float4 *>(&h) + lane, reinterpret_cast<const float4 *>(P.brec + s) + lane);
  else if (lane == 4) cp_async<8>(&base, &P.strut_off[s]);
}
__device__ __forceinline__ bool band_live(const BandRec &h) { return h.nA + h.nB > 0; }
__device__ __forceinline__ int rec_cnt(int lc) { return lc >> 16; }
__device__ __forceinline__ int rec_first(int lc) { return lc & 0xffff; }
// stage 2: loop entries of both rings
__device__ __forceinline__ void fetch_entries(const TriParams &P, WarpRing &w, const BandRec &h, int lane) {
  if (!band_live(h)) return;
  if (lane < rec_cnt(h.lAc)) cp_async<16>(&w.le[0][lane], P.loop + 2 * (int64_t)h.aA + rec_first(h.lAc) + lane);
  if (lane < rec_cnt(h.lBc)) cp_async<16>(&w.le[1][lane], P.loop + 2 * (int64_t)h.aB + rec_first(h.lBc) + lane);
}
// stage 3: the arc records of the entries (first MAXRA of each ring)
__device__ __forceinline__ void fetch_arcs(const TriParams &P, WarpRing &w, const BandRec &h, int lane) {
  if (!band_live(h)) return;
#pragma unroll
  for (int r = 0; r < 2; r++) {
    const int cnt = rec_cnt(r ? h.lBc : h.lAc);
    const ArcRec *arcs = P.arc + (r ? h.aB : h.aA);
    const int nq = (cnt < MAXRA ? cnt : MAXRA) * 3;
    for (int k = lane; k < nq; k += 32) {
      const int e = k / 3;
      cp_async<16>(reinterpret_cast<float4 *>(&w.arc[r][e]) + (k - 3 * e),
                   reinterpret_cast<const float4 *>(arcs + le_arc(w.le[r][e].arc_fwd)) + (k - 3 * e));
    }
    if (lane < nq / 3)   // the entries' start vertices (ids from the loop entries)
      cp_async<16>(&w.vq[r][lane], P.vert + 2 * (int64_t)(r ? h.pB : h.pA) + le_vid(w.le[r][lane].cum));
  }
}

struct RingRef {
  const ArcRec *arcs;
  const float4 *vs;
  float ox, oy, oz;
  int cnt;
  // the ring's entries in global memory (rings of more than MAXRE entries): 32-bit words,
  // entry e at gent + e * gst, arc_fwd at word 0, cum at word gco
  const uint32_t *gent;
  int gst, gco;
};

// entry e of ring r: the first MAXRE from shared memory, the rest from global memory
__device__ __forceinline__ void ring_entry(const WarpRing &w, int r, const RingRef &R, int e, uint32_t &af, int &cum) {
  if (e < MAXRE) {
    af = w.le[r][e].arc_fwd;
    cum = w.le[r][e].cum;
  } else {
    af = __ldg(R.gent + (int64_t)e * R.gst);
    cum = (int)__ldg(R.gent + (int64_t)e * R.gst + R.gco);
  }
}

__device__ __forceinline__ ArcRec lds_arc(const ArcRec *p) {
  const float4 *q = reinterpret_cast<const float4 *>(p);
  float4 x = q[0], y = q[1], z = q[2];
  ArcRec a;
  a.ids = __float_as_uint(x.x); a.t0 = x.y; a.dt = x.z; a.ox = x.w;
  a.oy = y.x; a.oz = y.y; a.ax = y.z; a.ay = y.w;
  a.az = z.x; a.bx = z.y; a.by = z.z; a.bz = z.w;
  return a;
}

// Eq. 12 interior point jj of an arc with N segments, translated by the node centre o.  The
// one formula of every emit path, every operation rounded as written, so the two bands and the
// hole fan that share an arc produce the same bits (watertight seams).
__device__ __forceinline__ f3 arc_pt(const ArcRec &A, int N, int jj, float ox, float oy, float oz) {
  float t = __fmaf_rn((float)jj, __fdividef(A.dt, (float)N), A.t0);
  t = __fmaf_rn(-LMM_TWO_PI_F, rintf(__fmul_rn(t, 1.0f / LMM_TWO_PI_F)), t);
  float sn, cs;
  __sincosf(t, &sn, &cs);
  return F3(__fadd_rn(ox, __fmaf_rn(A.ax, sn, __fmaf_rn(A.bx, cs, A.ox))),
            __fadd_rn(oy, __fmaf_rn(A.ay, sn, __fmaf_rn(A.by, cs, A.oy))),
            __fadd_rn(oz, __fmaf_rn(A.az, sn, __fmaf_rn(A.bz, cs, A.oz))));
}

// Eq. 12 point idx of ring r, whose loop entry is e; endpoints are the shared vertices
__device__ __forceinline__ f3 ring_point_e(const WarpRing &w, int r, const RingRef &R, int e, int idx) {
  LoopRec L;
  ring_entry(w, r, R, e, L.arc_fwd, L.cum);
  const int N = le_N(L.arc_fwd), fwd = le_fwd(L.arc_fwd);
  const int j = idx - le_cum(L.cum);
  const int jj = fwd ? j : N - j;
  f3 p;
  if (jj == 0 || jj == N) {
    const uint32_t ids = e < MAXRA ? w.arc[r][e].ids : __ldg(&R.arcs[le_arc(L.arc_fwd)].ids);
    const int v = jj == 0 ? arc_vs(ids) : arc_ve(ids);
    const float4 q = __ldg(&R.vs[v]);
    p = F3(q.x, q.y, q.z);
  } else {
    const ArcRec A = e < MAXRA ? lds_arc(&w.arc[r][e]) : load_arc(R.arcs + le_arc(L.arc_fwd));
    return arc_pt(A, N, jj, R.ox, R.oy, R.oz);
  }
  return F3(__fadd_rn(R.ox, p.x), __fadd_rn(R.oy, p.y), __fadd_rn(R.oz, p.z));
}

// point idx of ring r, its entry found by a scan of the entry starts (windowed bands, holes)
__device__ __forceinline__ f3 ring_point(const WarpRing &w, int r, const RingRef &R, int idx) {
  int e = 0;
  if (R.cnt <= MAXRE) {
    for (int k = 1; k < R.cnt; k++) e += (le_cum(w.le[r][k].cum) <= idx) ? 1 : 0;
  } else {   // long ring (spilled nodes): last entry starting at or before idx, binary search
    int lo = 0, hi = R.cnt - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (le_cum((int)__ldg(R.gent + (int64_t)mid * R.gst + R.gco)) <= idx) lo = mid; else hi = mid - 1;
    }
    e = lo;
  }
  return ring_point_e(w, r, R, e, idx);
}

// Eq. 12 interior formula (entry and arc cached); entry start points are overwritten with
// the shared vertices afterwards
__device__ __forceinline__ f3 ring_point_formula(const WarpRing &w, int r, const RingRef &R, int e, int idx) {
  const LoopRec L = w.le[r][e];
  const int N = le_N(L.arc_fwd), fwd = le_fwd(L.arc_fwd);
  const int j = idx - le_cum(L.cum);
  const int jj = fwd ? j : N - j;
  const ArcRec A = lds_arc(&w.arc[r][e]);
  return arc_pt(A, N, jj, R.ox, R.oy, R.oz);
}

__device__ __forceinline__ void put_point(const Pts &pt, int k, f3 p) { pt.xy[k] = make_float2(p.x, p.y); pt.z[k] = p.z; }
__device__ __forceinline__ f3 get_point(const Pts &pt, int k) { const float2 q = pt.xy[k]; return F3(q.x, q.y, pt.z[k]); }

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

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void tri_words(f3 a, f3 b, f3 c, uint32_t *f) {
  f3 u = f_sub(b, a), v = f_sub(c, a);
  float nx = u.y * v.z - u.z * v.y, ny = u.z * v.x - u.x * v.z, nz = u.x * v.y - u.y * v.x;
  float l2 = nx * nx + ny * ny + nz * nz;
  float il = l2 > 0.0f ? rsqrt_approx(l2) : 0.0f;
  f[0] = __float_as_uint(nx * il); f[1] = __float_as_uint(ny * il); f[2] = __float_as_uint(nz * il);
  f[3] = __float_as_uint(a.x); f[4] = __float_as_uint(a.y); f[5] = __float_as_uint(a.z);
  f[6] = __float_as_uint(b.x); f[7] = __float_as_uint(b.y); f[8] = __float_as_uint(b.z);
  f[9] = __float_as_uint(c.x); f[10] = __float_as_uint(c.y); f[11] = __float_as_uint(c.z);
}

// records 2l (f) and 2l+1 (g) as 25 aligned words: f, then attribute 0 | g shifted by 16
__device__ __forceinline__ void put_first(uint32_t *d, const uint32_t *f) {
#pragma unroll
  for (int i = 0; i < 12; i++) d[i] = f[i];
}
__device__ __forceinline__ void put_second(uint32_t *d, const uint32_t *g) {
  d[12] = g[0] << 16;
#pragma unroll
  for (int i = 0; i < 11; i++) d[13 + i] = __funnelshift_r(g[i], g[i + 1], 16);
  d[24] = g[11] >> 16;
}

// staged group bytes [b0, b1) -> dst + [b0, b1), dst 16-byte aligned: 2-byte head up to the
// first 16-byte boundary and 2-byte tail through the LSU, the 16-byte-aligned body as one
// TMA bulk copy (cp.async.bulk.global.shared::cta) issued by lane 0 -- the body bypasses
// the L1/LSU path.  The staging buffer may be rewritten after stage_wait().
__device__ __forceinline__ void stage_wait(int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  __syncwarp();
}
__device__ __forceinline__ void flush_group(WarpRing &w, int b0, int b1, unsigned char *dst, int lane) {
  __syncwarp();
  const int v0 = (b0 + 15) >> 4, v1 = b1 >> 4;
  const uint16_t *s16 = reinterpret_cast<const uint16_t *>(w.stage);
  uint16_t *d16 = reinterpret_cast<uint16_t *>(dst);
  if (v0 <= v1) {
    if (v1 > v0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // staging writes -> async proxy
      __syncwarp();
      if (lane == 0) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(w.stage + v0);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                     ::"l"(dst + 16 * v0), "r"(sa), "r"(16 * (v1 - v0)) : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    }
    const int h = (v0 << 3) - (b0 >> 1);          // head half-words
    if (lane < h) d16[(b0 >> 1) + lane] = s16[(b0 >> 1) + lane];
    const int t0 = v1 << 3, tn = (b1 >> 1) - t0;  // tail half-words
    if (lane < tn) d16[t0 + lane] = s16[t0 + lane];
  } else {                                          // range inside one 16-byte unit
    const int n = (b1 - b0) >> 1;
    if (lane < n) d16[(b0 >> 1) + lane] = s16[(b0 >> 1) + lane];
  }
  __syncwarp();
}

// Whole-band emission.  Point cache layout: A_i at i (i = 0..nA, A_nA = A_0) and B_j at
// nA + 1 + j (j = 0..nB, B_j = ring-B point (j + kB) mod nB), so triangle positions need
// no wrapping.  The band's merge-bit words are held one per lane.
template <class Prefetch>
__device__ void emit_band_whole(const TriParams &P, WarpRing &w, const Pts &pt, const RingRef &RA, const RingRef &RB,
                                int64_t base, int nA, int nB, int kB, int qb, int qe, int64_t first,
                                unsigned char *out, int lane, Prefetch &prefetch) {
  const int oB = nA + 1;
  const int64_t w0 = base >> 5;
  const int nwd = (int)(((base + nA + nB - 1) >> 5) - w0 + 1);
  const uint32_t mword = lane < nwd ? __ldg(&P.mbits[w0 + lane]) : 0u;
  // entry start vertices (prefetched with the arcs)
  float4 vq[2];
#pragma unroll
  for (int r = 0; r < 2; r++) vq[r] = lane < (r ? RB.cnt : RA.cnt) ? w.vq[r][lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  {
    const int cA = (lane >= 1 && lane < RA.cnt) ? le_cum(w.le[0][lane].cum) : 0x7fffffff;
    const int cB = lane < RB.cnt ? nA + le_cum(w.le[1][lane].cum) : 0x7fffffff;
    int run = 0;   // entry starts (after ring A's first) below the current block
    for (int x = 0; x < nA + nB; x += 32) {
      const int k = x + lane;
      const unsigned dA = (unsigned)(cA - x), dB = (unsigned)(cB - x);
      const unsigned bits = (dA < 32u ? 1u << dA : 0u) | (dB < 32u ? 1u << dB : 0u);
      const unsigned M = __reduce_or_sync(0xffffffffu, bits);
      const int ec = run + __popc(M & ((2u << lane) - 1u));
      run += __popc(M);
      if (k < nA + nB) {
        if (ec < RA.cnt) {
          const f3 p = ring_point_formula(w, 0, RA, ec, k);
          put_point(pt, k, p);
          if (k == 0) put_point(pt, nA, p);
        } else {
          const int idx = k - nA;
          const f3 p = ring_point_formula(w, 1, RB, ec - RA.cnt, idx);
          const int jr = idx - kB + (idx < kB ? nB : 0);
          put_point(pt, oB + jr, p);
          if (jr == 0) put_point(pt, oB + nB, p);
        }
      }
    }
    __syncwarp();
    // entry start points are the shared meta-mesh vertices, bit for bit (watertight seams)
#pragma unroll
    for (int r = 0; r < 2; r++) {
      const RingRef &R = r ? RB : RA;
      if (lane < R.cnt) {
        const float4 q = vq[r];
        const f3 p = F3(R.ox + q.x, R.oy + q.y, R.oz + q.z);
        const int idx = le_cum(w.le[r][lane].cum);
        if (r == 0) {
          put_point(pt, idx, p);
          if (idx == 0) put_point(pt, nA, p);
        } else {
          const int jr = idx - kB + (idx < kB ? nB : 0);
          put_point(pt, oB + jr, p);
          if (jr == 0) put_point(pt, oB + nB, p);
        }
      }
    }
    __syncwarp();
  }
  prefetch(1);   // the ring data of this band is dead from here on
  const unsigned lt = (1u << lane) - 1u;
  int irun = qb == 0 ? 0 : merge_rank(P, base, base + qb);
  const int sb = (int)(base & 31);
  bool second = false;
  for (int gq = qb - (int)((base + qb - first) & 7); gq < qe; gq += GRP) {
    const int qa = gq + 2 * lane, qb2 = qa + 1;
    const int lo_q = gq > qb ? gq : qb;
    const int hi_q = gq + GRP < qe ? gq + GRP : qe;
    const bool whole = gq >= qb && gq + GRP <= qe;
    const bool va = whole ? lane < GRP / 2 : (qa >= lo_q && qa < hi_q);
    const bool vb = whole ? lane < GRP / 2 : (qb2 >= lo_q && qb2 < hi_q);
    // bit of step q: word (sb + q) >> 5 of the band's words, from the owning lane
    const int ba = sb + (va ? qa : 0), bb = sb + (vb ? qb2 : 0);
    const uint32_t wa = __shfl_sync(0xffffffffu, mword, ba >> 5), wb = __shfl_sync(0xffffffffu, mword, bb >> 5);
    const bool aa = va && ((wa >> (ba & 31)) & 1u);
    const bool ab = vb && ((wb >> (bb & 31)) & 1u);
    const unsigned ma = __ballot_sync(0xffffffffu, aa), mb = __ballot_sync(0xffffffffu, ab);
    const int ia = irun + __popc(ma & lt) + __popc(mb & lt);
    irun += __popc(ma) + __popc(mb);
    stage_wait(lane);
    if (va || vb) {
      // state before the lane's first valid step: A_i, B_j; each triangle (A_i, c, B_j)
      // advances one ring onto its new point c
      int i = ia, j = (va ? qa : qb2) - ia;
      f3 pA = get_point(pt, i), pB = get_point(pt, oB + j);
      uint32_t *d = reinterpret_cast<uint32_t *>(w.stage) + 25 * lane;   // records 2l, 2l+1
      if (va) {
        const f3 c = get_point(pt, aa ? i + 1 : oB + j + 1);
        uint32_t f[12];
        tri_words(pA, c, pB, f);
        put_first(d, f);
        if (aa) { pA = c; i++; } else { pB = c; j++; }
      }
      if (vb) {
        const f3 c = get_point(pt, ab ? i + 1 : oB + j + 1);
        uint32_t g[12];
        tri_words(pA, c, pB, g);
        put_second(d, g);
      }
    }
    if (whole) {   // a whole group: one bulk copy, no head or tail
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(w.stage);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                     ::"l"(out + (base + gq - first) * REC), "r"(sa), "n"(GRP * REC) : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    } else flush_group(w, (lo_q - gq) * REC, (hi_q - gq) * REC, out + (base + gq - first) * REC, lane);
    if (!second) { prefetch(2); second = true; }
  }
  if (!second) prefetch(2);
  prefetch(3);
}

template <class Prefetch>
__device__ void emit_band(const TriParams &P, WarpRing &w, const Pts &pt, const BandRec &H, int64_t base, int64_t first,
                          int64_t lo, int64_t hi, unsigned char *out, int lane, Prefetch prefetch) {
  // triangles [lo, hi) of the band; output record t at out + (t - first) * REC
  const int nA = H.nA, nB = H.nB, kB = H.kB;
  const int64_t ta = base > lo ? base : lo;
  const int64_t tb = base + nA + nB < hi ? base + nA + nB : hi;
  if (ta >= tb) { prefetch(0); prefetch(1); prefetch(2); prefetch(3); return; }
  RingRef RA, RB;
  RA.arcs = P.arc + H.aA;
  RA.vs = P.vert + 2 * (int64_t)H.pA;
  RA.ox = H.oax; RA.oy = H.oay; RA.oz = H.oaz; RA.cnt = rec_cnt(H.lAc);
  RA.gent = reinterpret_cast<const uint32_t *>(P.loop + 2 * (int64_t)H.aA + rec_first(H.lAc));
  RA.gst = 4; RA.gco = 3;
  RB.arcs = P.arc + H.aB;
  RB.vs = P.vert + 2 * (int64_t)H.pB;
  RB.ox = H.obx; RB.oy = H.oby; RB.oz = H.obz; RB.cnt = rec_cnt(H.lBc);
  RB.gent = reinterpret_cast<const uint32_t *>(P.loop + 2 * (int64_t)H.aB + rec_first(H.lBc));
  RB.gst = 4; RB.gco = 3;
  const int qb = (int)(ta - base), qe = (int)(tb - base);
  prefetch(0);
  if (nA + nB + 2 <= pt.cap && RA.cnt <= MAXRA && RB.cnt <= MAXRA) {
    emit_band_whole(P, w, pt, RA, RB, base, nA, nB, kB, qb, qe, first, out, lane, prefetch);
    return;
  }
  // windowed: the ring data stays in use to the end, the next band's stages follow it
  const unsigned lt = (1u << lane) - 1u;
  for (int q0 = qb, q1; q0 < qe; q0 = q1) {
    q1 = q0 - (int)((base + q0 - first) & 7) + pt.cap - 2;   // windows end on the 8-triangle grid
    q1 = q1 < qe ? q1 : qe;
    int i0 = 0, i1 = 0;
    if (lane == 0) i0 = merge_rank(P, base, base + q0);
    if (lane == 1) i1 = (q1 == nA + nB) ? nA : merge_rank(P, base, base + q1);
    i0 = __shfl_sync(0xffffffffu, i0, 0);
    i1 = __shfl_sync(0xffffffffu, i1, 1);
    const int j0 = q0 - i0, j1 = q1 - i1;
    const int na = i1 - i0 + 1;
    const int nb = j1 - j0 + 1;
    for (int k = lane; k < na + nb; k += 32) {
      const int r = k < na ? 0 : 1;
      const int kk = r ? k - na : k;
      const int n = r ? nB : nA;
      int idx = r ? j0 + kk + kB : i0 + kk;
      idx = idx >= n ? idx - n : idx;
      idx = idx >= n ? idx - n : idx;
      f3 p = r ? ring_point(w, 1, RB, idx) : ring_point(w, 0, RA, idx);
      put_point(pt, k, p);
    }
    __syncwarp();
    // the record of step q is the triangle (A_i, A_i+1, B_j) or (A_i, B_j+1, B_j)
    auto tri = [&](int q, int i, bool advA, uint32_t *f) {
      const int pa = i - i0, pb = na + (q - i - j0);
      const int pc = advA ? pa + 1 : pb + 1;
      tri_words(get_point(pt, pa), get_point(pt, pc), get_point(pt, pb), f);
    };
    int irun = i0;
    for (int gq = q0 - (int)((base + q0 - first) & 7); gq < q1; gq += GRP) {
      const int qa = gq + 2 * lane, qb2 = qa + 1;
      const int lo_q = gq > q0 ? gq : q0;
      const int hi_q = gq + GRP < q1 ? gq + GRP : q1;
      const bool va = qa >= lo_q && qa < hi_q, vb = qb2 >= lo_q && qb2 < hi_q;
      const int64_t ta2 = base + qa;
      const bool aa = va && ((__ldg(&P.mbits[ta2 >> 5]) >> (ta2 & 31)) & 1u);
      const bool ab = vb && ((__ldg(&P.mbits[(ta2 + 1) >> 5]) >> ((ta2 + 1) & 31)) & 1u);
      const unsigned ma = __ballot_sync(0xffffffffu, aa), mb = __ballot_sync(0xffffffffu, ab);
      const int ia = irun + __popc(ma & lt) + __popc(mb & lt);
      irun += __popc(ma) + __popc(mb);
      stage_wait(lane);
      if (va || vb) {
        uint32_t *d = reinterpret_cast<uint32_t *>(w.stage) + 25 * lane;
        uint32_t f[12];
        if (va) { tri(qa, ia, aa, f); put_first(d, f); }
        if (vb) { tri(qb2, ia + (aa ? 1 : 0), ab, f); put_second(d, f); }
      }
      if (gq >= q0 && gq + GRP <= q1) {   // a whole group: one bulk copy, no head or tail
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(w.stage);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                       ::"l"(out + (base + gq - first) * REC), "r"(sa), "n"(GRP * REC) : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
      } else flush_group(w, (lo_q - gq) * REC, (hi_q - gq) * REC, out + (base + gq - first) * REC, lane);
    }
    __syncwarp();
  }
  prefetch(1);
  prefetch(2);
  prefetch(3);
}

__device__ void emit_hole(const TriParams &P, WarpRing &w, const Pts &pt, int g, int64_t first, int64_t last,
                          unsigned char *out, int lane) {
  const int64_t hb = P.n_tri_band + P.hole_off[g];
  const int M = P.hole_M[g];
  const int64_t ta = hb > first ? hb : first;
  const int64_t tb = hb + M < last ? hb + M : last;
  if (ta >= tb) return;
  const int n = P.hole_node[g];
  const int64_t g0 = P.node_hole0[n];
  const int2 key = P.skey[n];
  const int2 H = P.hole_hdr[hbase(key) + (g - g0)];
  const float4 on = P.node[n];
  const float4 bp4 = P.hole_bp[g];
  const f3 bp = F3(on.x + bp4.x, on.y + bp4.y, on.z + bp4.z);
  RingRef RH;
  RH.arcs = P.arc + abase(key); RH.vs = P.vert + vbase(key);
  RH.ox = on.x; RH.oy = on.y; RH.oz = on.z; RH.cnt = H.y;
  // hole entries (arc_fwd, cum) in the loop-entry slots of ring 0 (the first MAXRE)
  const HoleEnt *he = P.hole_ent + hebase(key) + H.x;
  RH.gent = reinterpret_cast<const uint32_t *>(he);
  RH.gst = 2; RH.gco = 1;
  __syncwarp();
  if (lane < H.y) {
    HoleEnt E = he[lane];
    LoopRec L;
    L.arc_fwd = E.arc_fwd; L.phs = 0.0f; L.dph = 0.0f; L.cum = E.cum;
    w.le[0][lane] = L;
  }
  __syncwarp();
  {
    const int nq = (H.y < MAXRA ? H.y : MAXRA) * 3;
    float4 *dst = reinterpret_cast<float4 *>(w.arc[0]);
    for (int k = lane; k < nq; k += 32) dst[k] = __ldg(reinterpret_cast<const float4 *>(RH.arcs + le_arc(w.le[0][k / 3].arc_fwd)) + (k % 3));
  }
  __syncwarp();
  const int mb = (int)(ta - hb), me = (int)(tb - hb);
  for (int m0 = mb, m1; m0 < me; m0 = m1) {
    m1 = m0 - (int)((hb + m0 - first) & 7) + pt.cap - 2;   // windows end on the 8-triangle grid
    m1 = m1 < me ? m1 : me;
    for (int k = lane; k <= m1 - m0; k += 32) {
      int idx = m0 + k;
      put_point(pt, k, ring_point(w, 0, RH, idx >= M ? idx - M : idx));
    }
    __syncwarp();
    // fan triangles (b_project, P_m, P_m+1) in aligned groups, two records per lane, leaving
    // through the staging buffer like the band groups
    for (int gq = m0 - (int)((hb + m0 - first) & 7); gq < m1; gq += GRP) {
      const int qa = gq + 2 * lane, qb2 = qa + 1;
      const int lo_q = gq > m0 ? gq : m0;
      const int hi_q = gq + GRP < m1 ? gq + GRP : m1;
      const bool va = qa >= lo_q && qa < hi_q, vb = qb2 >= lo_q && qb2 < hi_q;
      stage_wait(lane);
      uint32_t *d = reinterpret_cast<uint32_t *>(w.stage) + 25 * lane;   // records 2l, 2l+1
      if (va) {
        uint32_t f[12];
        tri_words(bp, get_point(pt, qa - m0), get_point(pt, qa - m0 + 1), f);
        put_first(d, f);
      }
      if (vb) {
        uint32_t f[12];
        tri_words(bp, get_point(pt, qb2 - m0), get_point(pt, qb2 - m0 + 1), f);
        put_second(d, f);
      }
      flush_group(w, (lo_q - gq) * REC, (hi_q - gq) * REC, out + (hb + gq - first) * REC, lane);
    }
    __syncwarp();
  }
}

__device__ __forceinline__ unsigned mask_ge(int x) { return x >= 32 ? 0u : (x <= 0 ? 0xffffffffu : (0xffffffffu << x)); }
__device__ __forceinline__ unsigned mask_le(int x) { return x < 0 ? 0u : (x >= 31 ? 0xffffffffu : ((2u << x) - 1u)); }

struct NoPrefetch {
  __device__ void operator()(int) const {}
};
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }


// ---------------------------------------------------------------------------------
// CTA-window emission of the band region (bands short against the window: k_emit_span)
//
// A CTA owns the band triangles [T0, T1) of a span (T0 - first a multiple of GW, so every
// group of GW records starts on the 16-byte output grid) and walks its bands in windows:
// up to SNB whole bands (warp 0 reads their records lane-parallel, lane = band) whose points
// fit the CTA's point cache and whose loop entries fit SEC (thread = entry).  Every thread
// stages its entry's loop record, arc record and start vertex by cp.async and turns them
// into the Eq. 12 parameters and cache placement of the entry's points; the window's points
// are then computed flattened over the CTA (the entry of a point from a bitmap of entry
// starts), and every complete group of GW triangles -- whatever bands its records belong
// to -- is assembled by one warp (lane = 2 records; band = slot from a redux of band
// starts; ring positions from the prefix counts of the merge bits) and leaves as one TMA
// bulk copy from the warp's staging buffer.  The group that a window leaves incomplete
// waits for the next window: the points its records still need move to the front of the
// cache.  A band too large for a window goes through emit_band (warp 0).
// ---------------------------------------------------------------------------------
constexpr int SNB = 32;           // bands per window (warp 0 lanes)
constexpr int SEC = EMIT_T;       // loop entries per window (one per thread)
constexpr int SMW = 48;           // merge-bit / point-bitmap words per window
constexpr int SPCW_MAX = 1280;    // point cache of a CTA window (runtime-sized)
constexpr int SPAN_CTA = 16384;   // band triangles per CTA span (a multiple of GW)
enum { ACT_WINDOW = 0, ACT_DONE = 1, ACT_LONG = 2 };
#ifndef LMM_SPAN_MINB
#define LMM_SPAN_MINB 6
#endif

struct __align__(16) SpanSm {
  PtEnt ent[SEC];                     // raw arc (48) | start vertex (16) | loop entry (16), then the entry
  uint4 stage[EW][GW * REC / 16];     // per-warp staging buffers
  // per window (double-buffered: the current one and the one built ahead)
  int s_ta[2][SNB], s_XA[2][SNB], s_XB[2][SNB];   // band k: first record; A_i at XA + C(q), B_j at XB + q - C(q)
  uint32_t mw[2][SMW];                // merge bits of the window's records (bits before the window cleared)
  int mp[2][SMW];                     //   exclusive prefix popcounts
  long long wb0[2];                   // global word of mw[b][0]
  int w_ta0[2], w_tend[2], w_K[2], w_Pn[2], w_Ew[2];   // first record, end, bands, points, entries
  // the built window's bands, for its entry set-up
  int b_pos[SNB], b_flx[SNB], b_kB[SNB], b_nA[SNB], b_nB[SNB], b_e0[SNB], b_cntA[SNB], b_fA[SNB], b_fB[SNB];
  unsigned b_aA[SNB], b_aB[SNB], b_pA[SNB], b_pB[SNB];
  alignas(16) float b_c[SNB][6];      // node centres (doubles as the band path's record)
  uint8_t e_band[SEC];
  uint32_t bm[SMW];                   // flattened point p starts an entry
  int act, gnext;
};
static_assert(offsetof(SpanSm, ent) % 16 == 0 && offsetof(SpanSm, stage) % 16 == 0 && offsetof(SpanSm, b_c) % 16 == 0,
              "cp.async / bulk-copy operands are 16-byte aligned");
__host__ __device__ constexpr int span_bytes(int pcw) { return (int)((sizeof(SpanSm) + (size_t)pcw * 12 + 15) / 16 * 16); }

// staged bytes [b0, b1) of a group -> dst + [b0, b1) (dst 16-byte aligned), as flush_group
__device__ __forceinline__ void flush_stage(uint4 *stage, int b0, int b1, unsigned char *dst, int lane) {
  __syncwarp();
  const int v0 = (b0 + 15) >> 4, v1 = b1 >> 4;
  const uint16_t *s16 = reinterpret_cast<const uint16_t *>(stage);
  uint16_t *d16 = reinterpret_cast<uint16_t *>(dst);
  if (v0 <= v1) {
    if (v1 > v0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(stage + v0);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                     ::"l"(dst + 16 * v0), "r"(sa), "r"(16 * (v1 - v0)) : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    }
    const int h = (v0 << 3) - (b0 >> 1);
    if (lane < h) d16[(b0 >> 1) + lane] = s16[(b0 >> 1) + lane];
    const int t0 = v1 << 3, tn = (b1 >> 1) - t0;
    if (lane < tn) d16[t0 + lane] = s16[t0 + lane];
  } else {
    const int n = (b1 - b0) >> 1;
    if (lane < n) d16[(b0 >> 1) + lane] = s16[(b0 >> 1) + lane];
  }
  __syncwarp();
}

// a window as its groups read it (per warp, set once per window): band k's first record,
// XA and XB in lane k's registers
struct WinG {
  const uint32_t *mw;   // merge bits, bits before the window cleared
  const int *mp;        //   their exclusive prefix popcounts
  int bgo;              // bit of record q = q + bgo
  int lo, hi, nslot;    // records [lo, hi), bands
  int ta, XA, XB;       // lane k: band k
};

// records [max(g, lo), min(g + GW, hi)) of group g (relative to T0), by one warp; d = the lane's
// two records in the warp's staging buffer
__device__ __forceinline__ void cta_group(const WinG &W, const Pts &pt, uint4 *stage, uint32_t *d, unsigned char *dst, int g,
                                          int lane) {
  const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
  const int r0 = 2 * lane;
  const int q0 = g + r0, q1 = q0 + 1;
  const bool full = W.lo <= g && W.hi >= g + GW;
  const bool va = full || (q0 >= W.lo && q0 < W.hi), vb = full || (q1 >= W.lo && q1 < W.hi);
  const int bg = g + W.bgo;
  const int b0 = bg + r0, b1 = b0 + 1;
  const bool aa = va && ((W.mw[b0 >> 5] >> (b0 & 31)) & 1u);
  const bool ab = vb && ((W.mw[b1 >> 5] >> (b1 & 31)) & 1u);
  const unsigned ma = __ballot_sync(FULL, aa), mb = __ballot_sync(FULL, ab);
  const int Cg = W.mp[bg >> 5] + __popc(W.mw[bg >> 5] & ~mask_ge(bg & 31));
  const int I0 = Cg + __popc(ma & lt) + __popc(mb & lt), I1 = I0 + (aa ? 1 : 0);
  // bands: kg holds g; band starts inside (g, g + GW)
  const int kg = __popc(__ballot_sync(FULL, lane < W.nslot && W.ta <= g)) - 1;
  const int dp = W.ta - g;
  const bool inb = lane < W.nslot && dp > 0 && dp < GW;
  int XA0, XB0, XA1, XB1;
  if (__ballot_sync(FULL, inb) == 0u) {   // one band holds the whole group
    XA0 = XA1 = __shfl_sync(FULL, W.XA, kg & 31);
    XB0 = XB1 = __shfl_sync(FULL, W.XB, kg & 31);
  } else {
    const unsigned lo32 = __reduce_or_sync(FULL, inb && dp < 32 ? 1u << dp : 0u);
    const unsigned hi32 = __reduce_or_sync(FULL, inb && dp >= 32 ? 1u << (dp - 32) : 0u);
    const int k0 = kg + __popc(lo32 & mask_le(r0)) + __popc(hi32 & mask_le(r0 - 32));
    const int k1 = kg + __popc(lo32 & mask_le(r0 + 1)) + __popc(hi32 & mask_le(r0 - 31));
    XA0 = __shfl_sync(FULL, W.XA, k0 & 31); XB0 = __shfl_sync(FULL, W.XB, k0 & 31);
    XA1 = __shfl_sync(FULL, W.XA, k1 & 31); XB1 = __shfl_sync(FULL, W.XB, k1 & 31);
  }
  const int pa = XA0 + I0, pb = XB0 + q0 - I0;
  const int pa1 = XA1 + I1, pb1 = XB1 + q1 - I1;
  {
    uint32_t f[12];
    if (va) tri_words(get_point(pt, pa), get_point(pt, aa ? pa + 1 : pb + 1), get_point(pt, pb), f);
    stage_wait(lane);   // the warp's previous bulk copy has read the staging buffer
    if (va) put_first(d, f);
  }
  if (vb) {
    uint32_t f[12];
    tri_words(get_point(pt, pa1), get_point(pt, ab ? pa1 + 1 : pb1 + 1), get_point(pt, pb1), f);
    put_second(d, f);
  }
  if (full) {
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(stage);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(sa), "n"(GW * REC) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  } else {
    const int wlo = W.lo > g ? W.lo : g, whi = W.hi < g + GW ? W.hi : g + GW;
    flush_stage(stage, (wlo - g) * REC, (whi - g) * REC, dst, lane);
  }
}

__global__ void __launch_bounds__(EMIT_T, LMM_SPAN_MINB) k_emit_span(TriParams P, int64_t first, int64_t count, unsigned char *out,
                                                         int64_t nspan, int span, int pcw) {
  extern __shared__ __align__(128) unsigned char smem[];
  SpanSm &S = *reinterpret_cast<SpanSm *>(smem);
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int BIG = 0x3fffffff;
  Pts pt;
  pt.xy = reinterpret_cast<float2 *>(smem + sizeof(SpanSm));
  pt.z = reinterpret_cast<float *>(pt.xy + pcw);
  pt.cap = pcw;
  const int64_t last = first + count;
  const int64_t bend = last < P.n_tri_band ? last : P.n_tri_band;
  for (int64_t u = blockIdx.x; u < nspan; u += gridDim.x) {
    const int64_t T0 = first + u * span;
    const int64_t T1 = T0 + span < bend ? T0 + span : bend;
    int64_t snext = 0;   // warp 0: the next candidate band
    enum { B_OK, B_END, B_NOFIT };
    // warp 0: build the window of whole bands from snext into buffer wb -- slots, merge words,
    // band parameters -- and start the cp.async of its loop entries, arcs and start vertices
    auto build = [&](int wb) -> int {
      for (;;) {
        const int64_t c = snext + lane;
        int64_t b = INT64_MAX, e = INT64_MAX;
        if (c < P.S) { b = P.strut_off[c]; e = P.strut_off[c + 1]; }
        // the next candidates towards L2 for the build after this one
        if (lane < 16) prefetch_l2(P.brec + snext + 32 + 2 * lane);
        else if (lane < 19) prefetch_l2(P.strut_off + snext + 32 + 16 * (lane - 16));
        const unsigned stopm = __ballot_sync(FULL, b >= T1);
        const int nst = stopm ? __ffs(stopm) - 1 : 32;
        const bool live = lane < nst && e > b;
        const unsigned livem = __ballot_sync(FULL, live);
        if (!livem) {
          if (nst < 32) return B_END;   // every further band starts at or after T1
          snext += 32;
          continue;
        }
        int nA = 0, nB = 0, kB = 0, lAc = 0, lBc = 0;
        unsigned aA = 0u, aB = 0u, pA = 0u, pB = 0u;
        float4 x2 = make_float4(0.f, 0.f, 0.f, 0.f), x3 = x2;
        if (live) {
          const float4 *q = reinterpret_cast<const float4 *>(P.brec + c);
          const float4 x0 = __ldg(q), x1 = __ldg(q + 1);
          x2 = __ldg(q + 2); x3 = __ldg(q + 3);
          nA = __float_as_int(x0.x); nB = __float_as_int(x0.y); kB = __float_as_int(x0.z); lAc = __float_as_int(x0.w);
          lBc = __float_as_int(x1.x); aA = __float_as_uint(x1.y); aB = __float_as_uint(x1.z); pA = __float_as_uint(x1.w);
          pB = __float_as_uint(x2.x);
        }
        const int npts = live ? min(nA + nB + 2, 2047) : 0;
        const int nent = live ? min(rec_cnt(lAc) + rec_cnt(lBc), 255) : 0;
        int v = npts | (nent << 16);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, v, o);
          if (lane >= o) v += y;
        }
        const int cp = v & 0xffff, ce = v >> 16;
        const int rk = __popc(livem & lt);
        const bool fit = live && cp <= pcw && ce <= SEC && rk < SNB;
        const unsigned fitm = __ballot_sync(FULL, fit);
        if (!fitm) return B_NOFIT;
        const int lastf = 31 - __clz(fitm);
        const int pos = cp - npts;
        const int cex = ce - nent;
        int i0 = 0;
        if (fit && b < T0) i0 = merge_rank(P, b, T0);
        const int own = fit ? nA - i0 : 0;
        int ca = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, ca, o);
          if (lane >= o) ca += y;
        }
        const int cAn = ca - own;   // A-advances of the window before the band
        const int ta0 = __shfl_sync(FULL, (int)((b > T0 ? b : T0) - T0), __ffs(fitm) - 1);
        if (fit) {
          const int ta = (int)((b > T0 ? b : T0) - T0);
          S.s_ta[wb][rk] = ta;
          S.s_XA[wb][rk] = pos + i0 - cAn;
          S.s_XB[wb][rk] = pos + nA + 1 + (b < T0 ? (int)(T0 - b) - i0 : 0) - ta + cAn;
          S.b_pos[rk] = pos; S.b_flx[rk] = cp - npts - 2 * rk; S.b_kB[rk] = kB; S.b_nA[rk] = nA; S.b_nB[rk] = nB;
          S.b_e0[rk] = cex; S.b_cntA[rk] = rec_cnt(lAc); S.b_fA[rk] = rec_first(lAc); S.b_fB[rk] = rec_first(lBc);
          S.b_aA[rk] = aA; S.b_aB[rk] = aB; S.b_pA[rk] = pA; S.b_pB[rk] = pB;
          S.b_c[rk][0] = x2.y; S.b_c[rk][1] = x2.z; S.b_c[rk][2] = x2.w;
          S.b_c[rk][3] = x3.x; S.b_c[rk][4] = x3.y; S.b_c[rk][5] = x3.z;
          for (int x = 0; x < nent; x++) S.e_band[cex + x] = (uint8_t)rk;
        }
        const int K = __popc(fitm);
        const int Ew = __shfl_sync(FULL, ce, lastf);
        int tend;
        {
          const int64_t el = __shfl_sync(FULL, e, lastf);
          tend = (int)((el < T1 ? el : T1) - T0);
        }
        snext += lastf + 1;
        // merge bits of the window's records (bits before ta0 cleared) and their prefix counts,
        // from the word of its first group
        const int g0 = ta0 & ~(GW - 1);
        const long long wb0 = (T0 + g0) >> 5;
        const long long wl = (T0 + tend - 1) >> 5;
        uint32_t mwv[2];
#pragma unroll
        for (int r = 0; r < 2; r++) {
          const int i = lane + 32 * r;
          uint32_t m = wb0 + i <= wl ? __ldg(&P.mbits[wb0 + i]) : 0u;
          const long long cut = T0 + ta0 - 32 * (wb0 + i);
          if (cut >= 32) m = 0u;
          else if (cut > 0) m &= 0xffffffffu << cut;
          mwv[r] = m;
        }
        int x0 = __popc(mwv[0]), x1 = __popc(mwv[1]);
        const int s0 = x0, s1 = x1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y0 = __shfl_up_sync(FULL, x0, o), y1 = __shfl_up_sync(FULL, x1, o);
          if (lane >= o) { x0 += y0; x1 += y1; }
        }
        const int tot0 = __shfl_sync(FULL, x0, 31);
        if (lane < SMW) { S.mw[wb][lane] = mwv[0]; S.mp[wb][lane] = x0 - s0; }
        if (lane + 32 < SMW) { S.mw[wb][lane + 32] = mwv[1]; S.mp[wb][lane + 32] = tot0 + x1 - s1; }
        if (lane == 0) { S.wb0[wb] = wb0; S.w_ta0[wb] = ta0; S.w_tend[wb] = tend; S.w_K[wb] = K; }
        {
          const int Pn = __shfl_sync(FULL, cp, lastf) - 2 * K;
          if (lane == 0) { S.w_Pn[wb] = Pn; S.w_Ew[wb] = Ew; }
        }
        __syncwarp();
        // stage the loop entries, then (once they are in) their arcs and start vertices
        for (int e2 = lane; e2 < Ew; e2 += 32) {
          const int k = S.e_band[e2];
          const int x = e2 - S.b_e0[k];
          const bool rB = x >= S.b_cntA[k];
          const unsigned ab = rB ? S.b_aB[k] : S.b_aA[k];
          cp_async<16>(reinterpret_cast<float4 *>(&S.ent[e2]) + 4,
                       P.loop + 2 * (int64_t)ab + (rB ? S.b_fB[k] + x - S.b_cntA[k] : S.b_fA[k] + x));
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        for (int e2 = lane; e2 < Ew; e2 += 32) {
          const int k = S.e_band[e2];
          const bool rB = e2 - S.b_e0[k] >= S.b_cntA[k];
          float4 *slot = reinterpret_cast<float4 *>(&S.ent[e2]);
          const LoopRec L = *reinterpret_cast<const LoopRec *>(slot + 4);
          const float4 *ar = reinterpret_cast<const float4 *>(P.arc + (rB ? S.b_aB[k] : S.b_aA[k]) + le_arc(L.arc_fwd));
          cp_async<16>(slot, ar);
          cp_async<16>(slot + 1, ar + 1);
          cp_async<16>(slot + 2, ar + 2);
          cp_async<16>(slot + 3, P.vert + 2 * (int64_t)(rB ? S.b_pB[k] : S.b_pA[k]) + le_vid(L.cum));
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        return B_OK;
      }
    };
    // warp 0, no window built ahead: bands too large for a window go through the band path
    // until a window is built or the span is done; returns the action for all warps
    auto settle = [&](int st, int wb) -> int {
      for (;;) {
        if (st == B_OK) return ACT_WINDOW;
        if (st == B_END) return ACT_DONE;
        int64_t sl;
        {
          const int64_t c = snext + lane;
          int64_t b = INT64_MAX, e = INT64_MAX;
          if (c < P.S) { b = P.strut_off[c]; e = P.strut_off[c + 1]; }
          const unsigned livem = __ballot_sync(FULL, b < T1 && e > b);
          sl = snext + __ffs(livem) - 1;   // a live band exists (NOFIT)
        }
        WarpRing &w = *reinterpret_cast<WarpRing *>(&S.ent[0]);
        BandRec &lrec = *reinterpret_cast<BandRec *>(&S.b_c[0][0]);
        long long &lbase = *reinterpret_cast<long long *>(&S.b_pos[0]);
        stage_wait(lane);
        fetch_rec(P, (int)sl, lrec, lbase, lane);
        cp_async_wait_warp();
        fetch_entries(P, w, lrec, lane);
        cp_async_wait_warp();
        fetch_arcs(P, w, lrec, lane);
        cp_async_wait_warp();
        emit_band(P, w, pt, lrec, lbase, first, T0, T1, out, lane, NoPrefetch());
        stage_wait(lane);
        __syncwarp();
        snext = sl + 1;
        st = build(wb);
      }
    };
    int wb = 0;
    if (warp == 0) {
      snext = P.cmap[T0 / TPC];
      for (;;) {
        const int64_t c = snext + 1 + lane;
        const unsigned m = __ballot_sync(FULL, c < P.S && P.strut_off[c] <= T0);
        snext += __popc(m);
        if (m != FULL) break;
      }
      const int act = settle(build(0), 0);
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      if (lane == 0) S.act = act;
      if (lane < SMW) S.bm[lane] = 0u;
      if (lane + 32 < SMW) S.bm[lane + 32] = 0u;
    }
    __syncthreads();
    while (S.act == ACT_WINDOW) {
      const int Ew = S.w_Ew[wb], Pn = S.w_Pn[wb];
      // ======== the window's entries (thread = entry): Eq. 12 parameters, point placement ========
      float4 vq = make_float4(0.f, 0.f, 0.f, 0.f);
      if (tid < Ew) {
        const int k = S.e_band[tid];
        const bool rB = tid - S.b_e0[k] >= S.b_cntA[k];
        const float4 *slot = reinterpret_cast<const float4 *>(&S.ent[tid]);
        const LoopRec L = *reinterpret_cast<const LoopRec *>(slot + 4);
        const ArcRec A = lds_arc(reinterpret_cast<const ArcRec *>(slot));
        vq = slot[3];
        const int N = le_N(L.arc_fwd), ci = le_cum(L.cum);
        const int pos = S.b_pos[k], nA = S.b_nA[k], nB = S.b_nB[k], kB = S.b_kB[k];
        PtEnt E;
        E.t0 = A.t0; E.dq = __fdividef(A.dt, (float)N);
        E.ox = A.ox; E.oy = A.oy; E.oz = A.oz; E.ax = A.ax; E.ay = A.ay; E.az = A.az;
        E.bx = A.bx; E.by = A.by; E.bz = A.bz;
        E.cx = S.b_c[k][rB ? 3 : 0]; E.cy = S.b_c[k][rB ? 4 : 1]; E.cz = S.b_c[k][rB ? 5 : 2];
        E.nf = N | (le_fwd(L.arc_fwd) << 16);
        if (!rB) {
          E.P0 = pos + ci; E.wj = BIG; E.dupj = ci == 0 ? 0 : -1; E.off = nA;
        } else {
          const int bs = pos + nA + 1;
          E.off = nB;
          if (ci >= kB) { E.P0 = bs + ci - kB; E.wj = BIG; E.dupj = ci == kB ? 0 : -1; }
          else {
            E.P0 = bs + ci - kB + nB;
            if (ci + N > kB) { E.wj = kB - ci; E.dupj = kB - ci; } else { E.wj = BIG; E.dupj = -1; }
          }
        }
        const int est = S.b_flx[k] + (rB ? nA : 0) + ci;
        E.pad = est;
        S.ent[tid] = E;
        atomicOr(&S.bm[est >> 5], 1u << (est & 31));
      }
      __syncthreads();
      // ======== the window's points, flattened (entry of point p from the entry-start bitmap) ========
      {
        // exclusive prefix popcounts of the bitmap, per warp in registers (lane i: words i, i + 32)
        const uint32_t m0 = lane < SMW ? S.bm[lane] : 0u, m1 = lane + 32 < SMW ? S.bm[lane + 32] : 0u;
        int x0 = __popc(m0), x1 = __popc(m1);
        const int s0 = x0, s1 = x1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y0 = __shfl_up_sync(FULL, x0, o), y1 = __shfl_up_sync(FULL, x1, o);
          if (lane >= o) { x0 += y0; x1 += y1; }
        }
        x0 -= s0;
        x1 += __shfl_sync(FULL, x0 + s0, 31) - s1;
        for (int pb = warp * 32; pb < Pn; pb += EMIT_T) {
          const int p = pb + lane;
          const int wd = p >> 5;   // warp-uniform
          const int bpv = __shfl_sync(FULL, wd < 32 ? x0 : x1, wd & 31);
          const uint32_t bmv = __shfl_sync(FULL, wd < 32 ? m0 : m1, wd & 31);
          if (p < Pn) {
            const int e = bpv + __popc(bmv & mask_le(lane)) - 1;
            const float4 *q = reinterpret_cast<const float4 *>(&S.ent[e]);
            const float4 e0 = q[0], e1 = q[1], e2 = q[2], e3 = q[3];
            const int4 e4 = reinterpret_cast<const int4 *>(q)[4];   // wj dupj off est
            const int j = p - e4.w;
            const int nf = __float_as_int(e3.z), P0 = __float_as_int(e3.w);
            const int N = nf & 0xffff;
            const int jj = (nf >> 16) ? j : N - j;
            float t = __fmaf_rn((float)jj, e0.y, e0.x);
            t = __fmaf_rn(-LMM_TWO_PI_F, rintf(__fmul_rn(t, 1.0f / LMM_TWO_PI_F)), t);
            float sn, cs;
            __sincosf(t, &sn, &cs);
            // e0 = t0 dq ox oy, e1 = oz ax ay az, e2 = bx by bz cx, e3 = cy cz nf P0 (PtEnt)
            const f3 pq = F3(__fadd_rn(e2.w, __fmaf_rn(e1.y, sn, __fmaf_rn(e2.x, cs, e0.z))),
                             __fadd_rn(e3.x, __fmaf_rn(e1.z, sn, __fmaf_rn(e2.y, cs, e0.w))),
                             __fadd_rn(e3.y, __fmaf_rn(e1.w, sn, __fmaf_rn(e2.z, cs, e1.x))));
            const int ps = P0 + j - (j >= e4.x ? e4.z : 0);
            put_point(pt, ps, pq);
            if (j == e4.y) put_point(pt, ps + e4.z, pq);
          }
        }
      }
      __syncthreads();
      // entry start points are the shared meta-mesh vertices, bit for bit (watertight seams)
      if (tid < Ew) {
        const PtEnt &E = S.ent[tid];
        const f3 q = F3(__fadd_rn(E.cx, vq.x), __fadd_rn(E.cy, vq.y), __fadd_rn(E.cz, vq.z));
        put_point(pt, E.P0, q);
        if (E.dupj == 0) put_point(pt, E.P0 + E.off, q);
      }
      if (tid == 0) S.gnext = 0;
      __syncthreads();
      // ======== the window's groups (first and last partial): warp 0 first builds the next
      // window and starts its fetches; the groups are taken from a counter ========
      {
        WinG W;
        W.mw = S.mw[wb]; W.mp = S.mp[wb];
        W.bgo = (int)(T0 - 32 * S.wb0[wb]);
        W.lo = S.w_ta0[wb]; W.hi = S.w_tend[wb]; W.nslot = S.w_K[wb];
        W.ta = lane < W.nslot ? S.s_ta[wb][lane] : BIG;
        W.XA = S.s_XA[wb][lane]; W.XB = S.s_XB[wb][lane];
        const int g0 = W.lo & ~(GW - 1);
        const int ng = (W.hi - g0 + GW - 1) / GW;
        uint4 *stage = S.stage[warp];
        uint32_t *d = reinterpret_cast<uint32_t *>(stage) + 25 * lane;
        unsigned char *dst0 = out + (T0 + g0 - first) * REC;
        if (warp == 0) {
          if (lane < SMW) S.bm[lane] = 0u;
          if (lane + 32 < SMW) S.bm[lane + 32] = 0u;
          // (a band too large for a window waits for the barrier: the band path uses the point cache)
          const int st = build(wb ^ 1);
          if (lane == 0) S.act = st == B_OK ? ACT_WINDOW : (st == B_END ? ACT_DONE : ACT_LONG);
        }
        const unsigned gna = (unsigned)__cvta_generic_to_shared(&S.gnext);
        for (;;) {
          int m = 0;
          if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(m) : "r"(gna) : "memory");
          m = __shfl_sync(FULL, m, 0);
          if (m >= ng) break;
          cta_group(W, pt, stage, d, dst0 + (int64_t)m * GW * REC, g0 + m * GW, lane);
        }
        if (warp == 0) asm volatile("cp.async.wait_all;\n" ::: "memory");   // the next window's entry data
      }
      __syncthreads();
      wb ^= 1;
      if (S.act == ACT_LONG) {
        if (warp == 0) {
          const int act = settle(B_NOFIT, wb);
          asm volatile("cp.async.wait_all;\n" ::: "memory");
          if (lane == 0) S.act = act;
          if (lane < SMW) S.bm[lane] = 0u;
          if (lane + 32 < SMW) S.bm[lane + 32] = 0u;
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// units: bands [s0, s1) then holes [g0, g1) intersecting [first, last)
__global__ void __launch_bounds__(EMIT_T, LMM_EMIT_BAND_MINB) k_emit(TriParams P, int64_t first, int64_t count, unsigned char *out,
                                                 int64_t s0, int64_t s1, int64_t g0, int64_t g1, int pcap) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ BandRec rec[EW][2];
  __shared__ long long rbase[EW][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wbase = smem + (size_t)warp * ring_bytes(pcap);
  WarpRing &w = *reinterpret_cast<WarpRing *>(wbase);
  Pts pt;
  pt.xy = reinterpret_cast<float2 *>(wbase + sizeof(WarpRing));
  pt.z = reinterpret_cast<float *>(pt.xy + pcap);
  pt.cap = pcap;
  const int64_t last = first + count;
  const int64_t gw = (int64_t)blockIdx.x * EW + warp, nw = (int64_t)gridDim.x * EW;
  const int64_t nb = s1 - s0, nh = g1 - g0;
  // band u+nw: record at band u's start, loop entries after band u's points, arc records
  // after its first group (three dependent stages overlapped with band u)
  int cb = 0;
  if (gw < nb) {   // first band: all stages up front
    fetch_rec(P, (int)(s0 + gw), rec[warp][0], rbase[warp][0], lane);
    cp_async_wait_warp();
    fetch_entries(P, w, rec[warp][0], lane);
    cp_async_wait_warp();
    fetch_arcs(P, w, rec[warp][0], lane);
    cp_async_wait_warp();
  }
  for (int64_t u = gw; u < nb + nh; u += nw) {
    if (u < nb) {
      const bool more = u + nw < nb;
      BandRec &nx = rec[warp][cb ^ 1];
      emit_band(P, w, pt, rec[warp][cb], rbase[warp][cb], first, first, last, out, lane, [&](int stage) {
        if (stage == 0) {
          if (more) fetch_rec(P, (int)(s0 + u + nw), nx, rbase[warp][cb ^ 1], lane);
          return;
        }
        if (!more) return;
        cp_async_wait_warp();
        if (stage == 1) fetch_entries(P, w, nx, lane);
        else if (stage == 2) fetch_arcs(P, w, nx, lane);
      });
      cp_async_wait_warp();
      cb ^= 1;
    } else emit_hole(P, w, pt, (int)(g0 + u - nb), first, last, out, lane);
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

TriParams make_params(lmm_ctx *c) {
  TriParams P;
  P.node = (const float4 *)c->node.p;
  P.csr_off = (const int *)c->csr_off.p;
  P.skey = (const int2 *)c->skey.p;
  P.csr_ent = (const int2 *)c->csr_ent.p;
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
  P.brec = (BandRec *)c->brec.p;
  P.node_mask = c->has_node_mask ? (const uint8_t *)c->node_mask.p : nullptr;
  P.strut_mask = c->has_strut_mask ? (const uint8_t *)c->strut_mask.p : nullptr;
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
  if ((rc = dev_alloc(c->ring_n, sizeof(int) * (2 * S + 1)))) return rc;
  const int T = 256;
  TriParams P = make_params(c);
  {
    KTimer t(c, LMM_K_COUNT);
    if (S) {
      (c->n_launch++), k_ring_count<<<(unsigned)((2 * S + T - 1) / T), T, 0, c->stream>>>(P, 2 * S, (int *)c->ring_n.p);
      (c->n_launch++), k_band_count<<<(unsigned)((S + T - 1) / T), T, 0, c->stream>>>(P, (const int *)c->ring_n.p);
    }
    if (N) (c->n_launch++), k_node_nholes<<<(unsigned)((N + T - 1) / T), T, 0, c->stream>>>((const int4 *)c->node_hdr.p, N, c->has_node_mask ? (const uint8_t *)c->node_mask.p : nullptr, (int *)c->node_hole0.p);
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
  if ((rc = dev_alloc(c->brec, sizeof(BandRec) * (S + 1)))) return rc;
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

// the band path of k_emit for [first, last) (bands grid-strided per warp, then holes): s0/s1
// = bands, g0/g1 = holes intersecting the range (from the chunk map)
static int launch_band_path(lmm_ctx *c, const TriParams &P, int64_t first, int64_t count, void *out_dev,
                            cudaStream_t st, bool bands) {
  int pcap = PCAP_MIN;
  {
    const int64_t live = c->S > 0 ? c->S : 1;
    const double mean = (double)c->n_tri_band / (double)live;
    while (pcap < PCAP_MAX && mean + 2.0 > pcap - 4) pcap = pcap + 160 < PCAP_MAX ? pcap + 160 : PCAP_MAX;
    if (const char *ev = getenv("LMM_PCAP")) {   // tuning override: PCAP_MIN + 16 k (< PCAP_MAX) or PCAP_MAX
      const int v = atoi(ev);
      if (v == PCAP_MAX || (v >= PCAP_MIN && v < PCAP_MAX && (v - PCAP_MIN) % 16 == 0)) pcap = v;
    }
  }
  const size_t smem = (size_t)ring_bytes(pcap) * EW;
  if (!c->emit_attr_set) {
    CUDA_TRY(cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_bytes(PCAP_MAX) * EW));
    CUDA_TRY(cudaFuncSetAttribute(k_emit_span, cudaFuncAttributeMaxDynamicSharedMemorySize, span_bytes(SPCW_MAX)));
    c->emit_attr_set = true;
  }
  int &occ = c->emit_occ[pcap == PCAP_MAX ? 31 : (pcap - PCAP_MIN) / 16];   // one slot per cache size
  if (occ == 0) {
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit, EMIT_T, smem));
    if (occ < 1) occ = 1;
  }
  const int64_t last = first + count;
  const int64_t nch = (c->n_tri + TPC - 1) / TPC;
  int64_t s0 = c->S, s1 = c->S, g0 = c->H, g1 = c->H;
  if (!c->pinned_scalar) CUDA_TRY(cudaMallocHost((void **)&c->pinned_scalar, 64));
  int *hm = (int *)(c->pinned_scalar + 2);
  const int64_t ca = first / TPC, cn = (last - 1) / TPC + 1;
  CUDA_TRY(cudaMemcpyAsync(hm, (int *)c->cmap.p + ca, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (cn < nch) CUDA_TRY(cudaMemcpyAsync(hm + 1, (int *)c->cmap.p + cn, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t cna = cn * TPC;
  if (bands && first < c->n_tri_band) {
    s0 = hm[0];
    s1 = (cn < nch && cna < c->n_tri_band) ? (int64_t)hm[1] + 1 : c->S;
  }
  if (last > c->n_tri_band) {
    g0 = (ca * TPC >= c->n_tri_band) ? hm[0] : 0;
    g1 = (cn < nch && cna >= c->n_tri_band) ? (int64_t)hm[1] + 1 : c->H;
  }
  if (s1 < s0) s1 = s0;
  if (g1 < g0) g1 = g0;
  const int64_t units = (s1 - s0) + (g1 - g0);
  if (units <= 0) return LMM_OK;
  int64_t grid = (int64_t)c->n_sm * occ;
  const int64_t need = (units + EW - 1) / EW;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  (c->n_launch++), k_emit<<<(unsigned)grid, EMIT_T, smem, st>>>(P, first, count, (unsigned char *)out_dev, s0, s1, g0, g1, pcap);
  CUDA_TRY(cudaGetLastError());
  return LMM_OK;
}

int triangulate_emit(lmm_ctx *c, int64_t first, int64_t count, void *out_dev, cudaStream_t st) {
  if (count <= 0) return LMM_OK;
  TriParams P = make_params(c);
  KTimer t(c, LMM_K_EMIT);
  // CTA windows when several mean bands fit a window (short bands: per-band work dominates the
  // band path), else the band path; hole fans always take the band path
  const int64_t live = c->S > 0 ? c->S : 1;
  const double mean = (double)c->n_tri_band / (double)live;
  int pcw = 768;
  if (const char *ev = getenv("LMM_SPCW")) { const int v = atoi(ev); if (v >= 256 && v <= SPCW_MAX) pcw = v; }
  int span = SPAN_CTA;
  if (const char *ev = getenv("LMM_SPAN")) { const int v = atoi(ev); if (v >= GW && v % GW == 0) span = v; }
  // (measured on octet100: CE 1e-2, 48 triangles per band: CTA windows 19.1 ms vs band path
  // 24.1 ms; CE 1e-3, 144 per band: 44.2 vs 42.8 ms)
  bool use_span = mean <= 100.0;
  if (const char *ev = getenv("LMM_EMIT_PATH")) use_span = atoi(ev) == 1 ? true : (atoi(ev) == 0 ? false : use_span);
  const int64_t last = first + count;
  if (first < c->n_tri_band) c->emit_path = use_span ? 1 : 0;
  if (!use_span || first >= c->n_tri_band) return launch_band_path(c, P, first, count, out_dev, st, true);
  if (!c->emit_attr_set) {
    CUDA_TRY(cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_bytes(PCAP_MAX) * EW));
    CUDA_TRY(cudaFuncSetAttribute(k_emit_span, cudaFuncAttributeMaxDynamicSharedMemorySize, span_bytes(SPCW_MAX)));
    c->emit_attr_set = true;
  }
  const size_t smem = (size_t)span_bytes(pcw);
  int &occ = c->emit_occ[40 + pcw / 128];
  if (occ == 0) {
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_emit_span, EMIT_T, smem));
    if (occ < 1) occ = 1;
  }
  const int64_t bend = last < c->n_tri_band ? last : c->n_tri_band;
  const int64_t nspan = (bend - first + span - 1) / span;
  int64_t grid = (int64_t)c->n_sm * occ;
  if (grid > nspan) grid = nspan;
  (c->n_launch++), k_emit_span<<<(unsigned)grid, EMIT_T, smem, st>>>(P, first, bend - first, (unsigned char *)out_dev, nspan, span, pcw);
  CUDA_TRY(cudaGetLastError());
  if (last > c->n_tri_band) return launch_band_path(c, P, first, count, out_dev, st, false);   // the hole fans
  return LMM_OK;
}
