// spill.cu -- meta-mesh of the nodes the degree-bucketed kernels cannot hold (PAPER.md
// Sec. 4.3.3: "the scheduler employs multiple warps to meta-mesh a single strut ... struts
// with more than 32 curves"): nodes of degree 32..63, and nodes whose junctions, vertex
// clusters, arcs or conic vertices exceed the fixed per-warp workspace of their bucket
// (JCAP / CCAP / ACAP / QCAP in metamesh.cu).
//
// One CTA of 256 threads (8 warps, synchronised through shared memory) owns one node at a
// time, persistent over the spill list.  The sides live in shared memory; junctions,
// clusters, arcs, loops and holes live in a per-CTA workspace in global memory that is
// carved per node from the counts of the previous phase, so no count is capped: when a node
// needs more than the workspace holds, the CTA reports the size it needs and the host
// reruns the spill list with a larger workspace.  Tie masks are 64-bit (sides 0..63).
//
// The steps and their binary32 arithmetic are those of metamesh.cu / the oracle
// (DESIGN.md Sec. 4 and Sec. 9): triples in lexicographic order with both roots,
// connected components of "within delta_c", conics walked through their vertices, the
// ambiguous-arc rule, loops by (phi, arc), hole contours.  Results go to a virtual slab slot
// (slab key (2S + voff, N + vn), reserved atomically in the overflow region behind the
// regular slabs) so that every consumer addresses the node's slabs exactly like a regular
// node's, through the slab key.
//
// COMPILED WITH -fmad=false.
#include "lmm_internal.h"
#include "mm_node.cuh"

namespace {
using namespace mm;

constexpr int ST = 256;          // threads per CTA
constexpr int NW = ST / 32;

struct SpillWS {                 // sides in shared memory; vertices in the global workspace
  float4 w4[LMM_MAXD_SPILL + 1];
  float4 wp[LMM_MAXD_SPILL + 1][2];
  float ux[LMM_MAXD_SPILL + 1], uy[LMM_MAXD_SPILL + 1], uz[LMM_MAXD_SPILL + 1];
  float s[LMM_MAXD_SPILL + 1], c[LMM_MAXD_SPILL + 1], L[LMM_MAXD_SPILL + 1], lim[LMM_MAXD_SPILL + 1];
  float asx[LMM_MAXD_SPILL + 1], asy[LMM_MAXD_SPILL + 1], asz[LMM_MAXD_SPILL + 1];
  float e1x[LMM_MAXD_SPILL + 1], e1y[LMM_MAXD_SPILL + 1], e1z[LMM_MAXD_SPILL + 1];
  float e2x[LMM_MAXD_SPILL + 1], e2y[LMM_MAXD_SPILL + 1], e2z[LMM_MAXD_SPILL + 1];
  int sign[LMM_MAXD_SPILL + 1];
  float *vx, *vy, *vz;
};

struct SpillParams {
  const float4 *node;
  const int *csr_off;
  const int2 *csr_ent;
  const int *list;
  const int *level;                // first vertex-resolution level of each listed node
  int n_list;
  int4 *node_hdr;
  int2 *skey;
  float4 *vert;
  ArcRec *arc;
  int2 *loop_hdr;
  LoopRec *loop;
  int2 *hole_hdr;
  HoleEnt *hole_ent;
  uint32_t *vmask_hi;
  int64_t S2, N, ovf_off, ovf_n;   // regular slab keys end at (S2, N); overflow reserve
  unsigned char *ws;
  int64_t wsb;                     // workspace bytes per CTA
  unsigned long long *ctl;         // [0] reservation (voff << 32 | vn), [1] workspace need, [2] unplaced nodes
};

__device__ __forceinline__ uint64_t bit64(int k) { return 1ull << k; }

// block-wide exclusive scan of one int per thread (all threads call)
__device__ int block_scan(int v, int *total, int *sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NW ? sm[lane] : 0, wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < NW) sm[lane] = wi - w;
    if (lane == NW - 1) sm[NW] = wi;
  }
  __syncthreads();
  const int r = sm[warp] + x - v;
  *total = sm[NW];
  __syncthreads();
  return r;
}

// lowest `key` over the block among threads with `pred` (INT_MAX if none), all threads call
__device__ int block_min(bool pred, int key, int *sm1) {
  if (threadIdx.x == 0) *sm1 = 0x7fffffff;
  __syncthreads();
  if (pred) atomicMin(sm1, key);
  __syncthreads();
  const int r = *sm1;
  __syncthreads();
  return r;
}

__device__ uint64_t block_or64(uint64_t v, unsigned long long *sm1) {
  if (threadIdx.x == 0) *sm1 = 0ull;
  __syncthreads();
  if (v) atomicOr(sm1, (unsigned long long)v);
  __syncthreads();
  const uint64_t r = *sm1;
  __syncthreads();
  return r;
}

// workspace carving: 16-byte aligned regions; false when the workspace is too small
struct Carve {
  unsigned char *base;
  int64_t cap, off = 0;
  bool ok = true;
  template <class T>
  __device__ T *take(int64_t n) {
    int64_t o = (off + 15) & ~(int64_t)15;
    off = o + n * (int64_t)sizeof(T);
    if (off > cap) ok = false;
    return reinterpret_cast<T *>(base + (ok ? o : 0));
  }
};

// validity tests with 64-bit exclusion masks, each side test rounded as hs(m, y) - tau
// (oracle valid_strut_pt / valid_sphere_junction / valid_sphere_pt)
__device__ bool sp_valid_strut(const Node<SpillWS> &nd, int d, uint64_t excl, f3 y, float tau, float delta) {
  if (tau < -delta) return false;
  for (int m = 1; m <= d; m++) {
    if ((excl >> m) & 1ull) continue;
    if (nd.hs(m, y) - tau > delta) return false;
  }
  return true;
}
__device__ bool sp_valid_sphere_junction(const Node<SpillWS> &nd, int d, uint64_t excl, f3 y, float delta) {
  for (int m = 1; m <= d; m++) {
    if ((excl >> m) & 1ull) continue;
    if (nd.hs(m, y) > delta) return false;
  }
  return true;
}
__device__ bool sp_valid_sphere_pt(const Node<SpillWS> &nd, int d, uint64_t excl, f3 y, float delta) {
  for (int m = 1; m <= d; m++) {
    if ((excl >> m) & 1ull) continue;
    if (nd.hs(m, y) > -delta) return false;
  }
  return true;
}

struct QEnt { int q; float t, us, uc; };          // a vertex on a conic
struct TEnt { float t0, dt, tmid; int vs, ve; };  // an interval of a conic

__device__ __forceinline__ int ceil_div_pos(int x, int k) { return x <= 0 ? 0 : (x + k - 1) / k; }

// the meta-mesh of node n; returns its status (0 = ok).  `need` > 0 on workspace shortage.
__device__ int spill_node(const SpillParams &P, SpillWS &ws, int n, int level, int64_t *need) {
  __shared__ int sm[NW + 2];
  __shared__ int sm1;
  __shared__ unsigned long long smo;
  __shared__ int lcnt[LMM_MAXD_SPILL + 1], lpos[LMM_MAXD_SPILL + 2], lfill[LMM_MAXD_SPILL + 1];
  __shared__ int hs_st, hs_nh, hs_nhe;
  __shared__ unsigned long long slot_sh;
  const int tid = threadIdx.x;
  const int off = P.csr_off[n];
  const int d = P.csr_off[n + 1] - off;
  const float4 on = P.node[n];
  const float R = on.w;
  // vertex resolution of this attempt: delta_c 2^level (reading R10, re-decision)
  const float delta = LMM_TOL_REL * R, dc = (LMM_CTOL_REL * R) * (float)(1 << level);
  const int ns = d + 1;
  Carve cv{P.ws + (int64_t)blockIdx.x * P.wsb, P.wsb};
  *need = 0;

  // ---- 1. sides ------------------------------------------------------------------------
  if (tid == 0) {
    ws.w4[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    ws.wp[0][0] = ws.wp[0][1] = make_float4(0.f, 0.f, 0.f, 0.f);
    ws.lim[0] = __int_as_float(0x7f800000);
  }
  bool bad = false;
  if (tid < d) {
    const int2 ent = P.csr_ent[off + tid];
    bad = !setup_side(ws, tid + 1, on, P.node[ent.y & 0x7fffffff], (int)((unsigned)ent.y >> 31));
  }
  if (__syncthreads_or(bad)) return LMM_NODE_STRUT;
  Node<SpillWS> nd{ws, d, R};

  // ---- 2. triple junctions, lexicographic (a<b<c), root-minor ---------------------------
  const int njmax = ns * (ns - 1) * (ns - 2) / 3;   // 2 C(ns, 3)
  float4 *jp = cv.take<float4>(njmax);
  uint32_t *jcode = cv.take<uint32_t>(njmax);
  int *lab = cv.take<int>(njmax);
  int *lab2 = cv.take<int>(njmax);
  if (!cv.ok) { *need = cv.off; return 0; }
  int nj = 0;
  const int ncube = ns * ns * ns;
  for (int base = 0; base < ncube; base += ST) {
    const int t = base + tid;
    const int a = t / (ns * ns), b = (t / ns) % ns, c = t % ns;
    bool v0 = false, v1 = false, sh = false;
    f3 y[2];
    float tau[2];
    if (t < ncube && a < b && b < c) {
      if (nd.junction_bf(a, b, c, y, tau)) {
        const uint64_t excl = bit64(a) | bit64(b) | bit64(c);
        v0 = a == 0 ? sp_valid_sphere_junction(nd, d, excl, y[0], delta) : sp_valid_strut(nd, d, excl, y[0], tau[0], delta);
        v1 = a == 0 ? sp_valid_sphere_junction(nd, d, excl, y[1], delta) : sp_valid_strut(nd, d, excl, y[1], tau[1], delta);
        // SHORT: a vertex beyond 0.45 L cos(beta) along any strut side of the triple
        const float lm = fminf(fminf(ws.lim[a], ws.lim[b]), ws.lim[c]);
        sh = (v0 && tau[0] > lm) || (v1 && tau[1] > lm);
      }
    }
    if (__syncthreads_or(sh)) return LMM_NODE_SHORT;
    int tot;
    const int pos = nj + block_scan((int)v0 + (int)v1, &tot, sm);
    const uint32_t code = (uint32_t)a | ((uint32_t)b << 6) | ((uint32_t)c << 12);
    if (v0) {
      jp[pos] = make_float4(y[0].x, y[0].y, y[0].z, 0.f);
      jcode[pos] = code | (fabsf(tau[0]) <= delta ? (1u << 19) : 0u);
    }
    if (v1) {
      const int p1 = pos + (v0 ? 1 : 0);
      jp[p1] = make_float4(y[1].x, y[1].y, y[1].z, 0.f);
      jcode[p1] = code | (1u << 18) | (fabsf(tau[1]) <= delta ? (1u << 19) : 0u);
    }
    nj += tot;
  }
  __syncthreads();

  // ---- 3. clustering: connected components of "junctions within delta_c (max-norm)" -----
  for (int j = tid; j < nj; j += ST) lab[j] = j;
  __syncthreads();
  for (;;) {
    bool changed = false;
    for (int j = tid; j < nj; j += ST) {
      const float4 pj = jp[j];
      int lj = lab[j];
      for (int k = 0; k < nj; k++) {
        const int lk = lab[k];
        if (lk < lj) {
          const float4 pk = jp[k];
          if (fabsf(pj.x - pk.x) <= dc && fabsf(pj.y - pk.y) <= dc && fabsf(pj.z - pk.z) <= dc) lj = lk;
        }
      }
      lab2[j] = lj;
      changed = changed || lj != lab[j];
    }
    __syncthreads();
    for (int j = tid; j < nj; j += ST) lab[j] = lab2[j];
    if (!__syncthreads_or(changed)) break;
  }
  // roots in index order -> cluster ids (lab2[root] = id)
  int nc = 0;
  for (int base = 0; base < nj; base += ST) {
    const int j = base + tid;
    const bool root = j < nj && lab[j] == j;
    int tot;
    const int id = nc + block_scan(root ? 1 : 0, &tot, sm);
    if (root) lab2[j] = id;
    nc += tot;
  }
  const int npairs = ns * (ns - 1) / 2;
  const int vcap = nc + npairs + 1;   // clusters, then at most one seam per side pair
  float *vx = cv.take<float>(vcap);
  float *vy = cv.take<float>(vcap);
  float *vz = cv.take<float>(vcap);
  unsigned long long *vmask = cv.take<unsigned long long>(vcap);
  if (!cv.ok) { *need = 2 * cv.off; return 0; }
  ws.vx = vx; ws.vy = vy; ws.vz = vz;   // (every thread writes the same pointers)
  __syncthreads();
  for (int j = tid; j < nj; j += ST)
    if (lab[j] == j) {
      const int id = lab2[j];
      const float4 q = jp[j];
      vx[id] = q.x; vy[id] = q.y; vz[id] = q.z; vmask[id] = 0ull;
    }
  __syncthreads();
  for (int j = tid; j < nj; j += ST) {
    const uint32_t code = jcode[j];
    uint64_t bits = bit64(code & 63u) | bit64((code >> 6) & 63u) | bit64((code >> 12) & 63u);
    if (code & (1u << 19)) bits |= 1ull;   // strut junction at tangent length ~0: on the sphere
    atomicOr(&vmask[lab2[lab[j]]], (unsigned long long)bits);
  }
  __syncthreads();
  int nv = nc;

  // ---- 4. arcs: every side pair's conic walked through its vertices ---------------------
  uint64_t um = 0ull;
  int qpart = 0;   // sum over clusters of C(popc, 2): vertices on conics, all pairs
  for (int q = tid; q < nc; q += ST) {
    const uint64_t m = vmask[q];
    um |= m;
    const int pc = __popcll(m);
    qpart += pc * (pc - 1) / 2;
  }
  um = block_or64(um, &smo);
  int qtot;
  block_scan(qpart, &qtot, sm);
  const int acap = npairs + qtot + 1;
  ArcRec *arcs = cv.take<ArcRec>(acap);
  float *atmid = cv.take<float>(acap);
  const int64_t scratch0 = cv.off;
  if (!cv.ok) { *need = 2 * cv.off; return 0; }
  int na = 0;
  for (int base = 0; base < ns * ns; base += ST) {
    const int t = base + tid;
    const int a = t / ns, b = t % ns;
    const bool pair = t < ns * ns && a < b;
    const uint64_t pm = pair ? (bit64(a) | bit64(b)) : 0ull;
    int nq = 0, e = 0, nint = 0;
    f3 o = F3(0.f, 0.f, 0.f), av = o, bv = o;
    if (pair) {
      for (int q = 0; q < nc; q++) nq += (vmask[q] & pm) == pm ? 1 : 0;
      const uint64_t strut_bits = a == 0 ? bit64(b) : pm;
      if (nq > 0 || !(um & strut_bits)) {
        bool conic_ok = true;
        if (a == 0) nd.circle(b, &o, &av, &bv);
        else conic_ok = nd.ellipse(a, b, &o, &av, &bv);
        if (!conic_ok) { if (nq > 0) e = LMM_NODE_CONIC; }
        else nint = nq == 0 ? 1 : nq;
      }
    }
    int ntot;
    const int ipos = block_scan(nint, &ntot, sm);
    cv.off = scratch0;
    QEnt *qe = cv.take<QEnt>(ntot + 1);
    TEnt *te = cv.take<TEnt>(ntot + 1);
    if (!cv.ok) { *need = 2 * cv.off; return 0; }
    int cnt = 0, closed = 0;
    if (nint > 0) {
      QEnt *Q = qe + ipos;
      TEnt *T = te + ipos;
      int k = 0;
      for (int q = 0; q < nc; q++) {
        if ((vmask[q] & pm) != pm) continue;
        float su, sc;
        const float tq = conic_t(o, av, bv, nd.V(q), &su, &sc);
        int j = k++;   // insertion by (t, cluster index)
        while (j > 0 && (tq < Q[j - 1].t || (tq == Q[j - 1].t && q < Q[j - 1].q))) { Q[j] = Q[j - 1]; j--; }
        Q[j].q = q; Q[j].t = tq; Q[j].us = su; Q[j].uc = sc;
      }
      for (int i = 0; i < nint; i++) {
        float ms, mc, t0, dt;
        int vs, ve;
        if (nq == 0) { ms = 0.0f; mc = 1.0f; t0 = 0.0f; dt = LMM_TWO_PI_F; vs = ve = -1; }
        else if (nq == 1) { ms = -Q[0].us; mc = -Q[0].uc; t0 = Q[0].t; dt = LMM_TWO_PI_F; vs = ve = Q[0].q; }
        else {
          const int j = i + 1 == nq ? 0 : i + 1;
          dt = j == 0 ? (Q[0].t + LMM_TWO_PI_F) - Q[nq - 1].t : Q[j].t - Q[i].t;
          if (!(dt > 0.0f)) { e = LMM_NODE_CHAIN; break; }
          const float sx = Q[i].us + Q[j].us, scc = Q[i].uc + Q[j].uc;
          const float l2 = sx * sx + scc * scc;
          if (l2 > 1e-6f) {
            const float l = sqrtf(l2);
            ms = sx / l; mc = scc / l;
            if (dt > LMM_PI_F) { ms = -ms; mc = -mc; }
          } else { ms = Q[i].uc; mc = -Q[i].us; }
          t0 = Q[i].t; vs = Q[i].q; ve = Q[j].q;
        }
        const f3 y = F3((o.x + av.x * ms) + bv.x * mc, (o.y + av.y * ms) + bv.y * mc, (o.z + av.z * ms) + bv.z * mc);
        const float tmid = a == 0 ? 0.0f : nd.h(a, y);
        const bool ok = a == 0 ? sp_valid_sphere_pt(nd, d, pm, y, delta) : sp_valid_strut(nd, d, pm, y, tmid, delta);
        if (!ok) continue;
        T[cnt].t0 = t0; T[cnt].dt = dt; T[cnt].tmid = tmid; T[cnt].vs = vs; T[cnt].ve = ve;
        if (vs < 0) closed = 1;
        cnt++;
      }
    }
    // the first error in pair order stops the node (the oracle walks pairs in that order)
    const int ep = block_min(e != 0, t, &sm1);
    if (ep != 0x7fffffff) {
      if (t == ep) sm[NW + 1] = e;
      __syncthreads();
      return sm[NW + 1];
    }
    int atot, ctot;
    const int apos = na + block_scan(cnt, &atot, sm);
    const int spos = nv + block_scan(closed, &ctot, sm);
    for (int i = 0; i < cnt; i++) {
      const TEnt &T = te[ipos + i];
      int vs = T.vs, ve = T.ve;
      if (vs < 0) {   // closed conic without vertex: its seam (t = 0) becomes a vertex
        vx[spos] = o.x + bv.x; vy[spos] = o.y + bv.y; vz[spos] = o.z + bv.z;
        vmask[spos] = pm;
        vs = ve = spos;
      }
      ArcRec &A = arcs[apos + i];
      A.ids = arc_ids(a, b, vs, ve);
      A.t0 = T.t0; A.dt = T.dt;
      A.ox = o.x; A.oy = o.y; A.oz = o.z;
      A.ax = av.x; A.ay = av.y; A.az = av.z;
      A.bx = bv.x; A.by = bv.y; A.bz = bv.z;
      atmid[apos + i] = T.tmid;
    }
    na += atot;
    nv += ctot;
    __syncthreads();
  }
  cv.off = scratch0;

  // ambiguous strut-strut arcs running under a strictly exposed hole lune are dropped
  // (R10): midpoint tangent length < delta and both end circles join its ends
  {
    int *keep = cv.take<int>(na + 1);
    if (!cv.ok) { *need = 2 * cv.off; return 0; }
    for (int i = tid; i < na; i += ST) {
      const uint32_t ids = arcs[i].ids;
      const int lo = arc_lo(ids), hi = arc_hi(ids), vs = arc_vs(ids), ve = arc_ve(ids);
      bool drop = false;
      if (lo > 0 && vs != ve && atmid[i] < delta) {
        bool ca = false, cb = false;
        for (int j = 0; j < na; j++) {
          const uint32_t jd = arcs[j].ids;
          if (arc_lo(jd) != 0) continue;
          const int js = arc_vs(jd), je = arc_ve(jd), jh = arc_hi(jd);
          if (!((js == vs && je == ve) || (js == ve && je == vs))) continue;
          if (jh == lo) ca = true;
          if (jh == hi) cb = true;
        }
        drop = ca && cb;
      }
      keep[i] = drop ? 0 : 1;
    }
    __syncthreads();
    int w = 0;
    for (int base = 0; base < na; base += ST) {
      const int i = base + tid;
      const bool kp = i < na && keep[i];
      ArcRec rec;
      if (kp) rec = arcs[i];
      int tot;
      const int pos = w + block_scan(kp ? 1 : 0, &tot, sm);
      if (kp) arcs[pos] = rec;
      w += tot;
      __syncthreads();
    }
    na = w;
  }
  cv.off = scratch0;
  // every junction vertex must carry an arc
  {
    int *used = cv.take<int>(nc + 1);
    if (!cv.ok) { *need = 2 * cv.off; return 0; }
    for (int q = tid; q < nc; q += ST) used[q] = 0;
    __syncthreads();
    for (int i = tid; i < na; i += ST) {
      const uint32_t ids = arcs[i].ids;
      if (arc_vs(ids) < nc) used[arc_vs(ids)] = 1;
      if (arc_ve(ids) < nc) used[arc_ve(ids)] = 1;
    }
    __syncthreads();
    bool miss = false;
    for (int q = tid; q < nc; q += ST) miss = miss || !used[q];
    if (__syncthreads_or(miss)) return LMM_NODE_UNREF;
  }
  if (nv > 1023) return LMM_NODE_ACAP;   // 10-bit vertex ids (never reached for degree <= 63)
  cv.off = scratch0;

  // ---- 5. arc loops per strut end, ordered by (phi, arc index) ---------------------------
  float *eps = cv.take<float>(2 * na + 2);
  float *edp = cv.take<float>(2 * na + 2);
  int *efw = cv.take<int>(2 * na + 2);
  int *lslot = cv.take<int>(2 * na + 2);
  LoopRec *le = cv.take<LoopRec>(2 * na + 2);
  if (!cv.ok) { *need = 2 * cv.off; return 0; }
  for (int i = tid; i < na; i += ST) {
    const ArcRec &A = arcs[i];
    const int lo = arc_lo(A.ids), hi = arc_hi(A.ids), avs = arc_vs(A.ids), ave = arc_ve(A.ids);
    for (int x = 0; x < 2; x++) {
      const int k = x ? hi : lo;
      if (k == 0) continue;
      const f3 as = nd.AS(k), e1 = nd.E1(k), e2 = nd.E2(k);
      const int fwd = f_dot(f_cross(F3(A.ax, A.ay, A.az), F3(A.bx, A.by, A.bz)), as) < 0.0f;
      const int vs = fwd ? avs : ave, ve = fwd ? ave : avs;
      const f3 Ps = nd.V(vs);
      float ps = atan2p(f_dot(Ps, e2), f_dot(Ps, e1));
      if (ps < 0.0f) ps += LMM_TWO_PI_F;
      float dph;
      if (vs == ve) dph = LMM_TWO_PI_F;
      else {
        const f3 Pe = nd.V(ve);
        float pe = atan2p(f_dot(Pe, e2), f_dot(Pe, e1));
        if (pe < 0.0f) pe += LMM_TWO_PI_F;
        dph = pe - ps;
        if (dph <= 0.0f) dph += LMM_TWO_PI_F;
      }
      eps[2 * i + x] = ps;
      edp[2 * i + x] = dph;
      efw[2 * i + x] = fwd;
    }
  }
  for (int k = tid; k <= d; k += ST) { lcnt[k] = 0; lfill[k] = 0; }
  __syncthreads();
  for (int i = tid; i < na; i += ST) {
    const uint32_t ids = arcs[i].ids;
    if (arc_lo(ids)) atomicAdd(&lcnt[arc_lo(ids)], 1);
    atomicAdd(&lcnt[arc_hi(ids)], 1);
  }
  __syncthreads();
  {
    int tot;
    const int ex = block_scan(tid <= d ? lcnt[tid] : 0, &tot, sm);   // d <= 63 < ST
    if (tid <= d) lpos[tid] = ex;
    if (tid == 0) lpos[d + 1] = tot;
  }
  __syncthreads();
  for (int i = tid; i < na; i += ST) {
    const uint32_t ids = arcs[i].ids;
    if (arc_lo(ids)) lslot[lpos[arc_lo(ids)] + atomicAdd(&lfill[arc_lo(ids)], 1)] = 2 * i;
    lslot[lpos[arc_hi(ids)] + atomicAdd(&lfill[arc_hi(ids)], 1)] = 2 * i + 1;
  }
  __syncthreads();
  int e = 0;
  const int k = tid + 1;
  if (k <= d) {
    const int cnt = lcnt[k], p0 = lpos[k];
    int *sl = lslot + p0;
    for (int i = 1; i < cnt; i++) {   // insertion by (phi, arc index)
      const int x = sl[i];
      const float px = eps[x];
      int j = i;
      while (j > 0 && (px < eps[sl[j - 1]] || (px == eps[sl[j - 1]] && x < sl[j - 1]))) { sl[j] = sl[j - 1]; j--; }
      sl[j] = x;
    }
    if (cnt == 0) e = LMM_NODE_EMPTY;
    else {
      float sum = 0.0f;
      for (int i = 0; i < cnt; i++) {
        const int sx = sl[i], sy = sl[i + 1 == cnt ? 0 : i + 1];
        const uint32_t X = arcs[sx >> 1].ids, Y = arcs[sy >> 1].ids;
        const int xe = efw[sx] ? arc_ve(X) : arc_vs(X);
        const int ys = efw[sy] ? arc_vs(Y) : arc_ve(Y);
        if (xe != ys) { e = LMM_NODE_CHAIN; break; }
        sum += edp[sx];
      }
      if (!e && fabsf(sum - LMM_TWO_PI_F) > 1e-3f) e = LMM_NODE_ANGLE;
    }
    if (!e) {
      float ph = eps[sl[0]];
      for (int i = 0; i < cnt; i++) {
        if (i > 0) ph = ph + edp[sl[i - 1]];
        LoopRec &L = le[p0 + i];
        const uint32_t aid = arcs[sl[i] >> 1].ids;
        L.arc_fwd = (uint32_t)(sl[i] >> 1) | ((uint32_t)efw[sl[i]] << 16);
        L.phs = ph;
        L.dph = edp[sl[i]];
        L.cum = (int32_t)((uint32_t)(efw[sl[i]] ? arc_vs(aid) : arc_ve(aid)) << LE_VID_SHIFT);
      }
    }
  }
  {
    const int ek = block_min(e != 0, k, &sm1);
    if (ek != 0x7fffffff) {
      if (k == ek) sm[NW + 1] = e;
      __syncthreads();
      return sm[NW + 1];
    }
  }
  const int nle = lpos[d + 1];

  // ---- 6. hole contours: cap arcs chained around the exposed sphere (one thread) ---------
  HoleEnt *he = cv.take<HoleEnt>(na + 1);
  int *hoff = cv.take<int>(na + 2);
  unsigned char *usd = cv.take<unsigned char>(na + 1);
  if (!cv.ok) { *need = 2 * cv.off; return 0; }
  if (tid == 0) {
    int st = 0, nh = 0, nhe = 0;
    for (int i = 0; i < na; i++) usd[i] = 0;
    for (int i = 0; i < na && !st; i++) {
      const uint32_t ai = arcs[i].ids;
      if (arc_lo(ai) != 0 || usd[i]) continue;
      hoff[nh++] = nhe;
      int cur = i;
      const int start_v = ws.sign[arc_hi(ai)] < 0 ? arc_vs(ai) : arc_ve(ai);
      for (;;) {
        usd[cur] = 1;
        const uint32_t ci = arcs[cur].ids;
        const int hf = ws.sign[arc_hi(ci)] < 0;
        he[nhe].arc_fwd = (uint32_t)cur | ((uint32_t)hf << 16);
        he[nhe].cum = 0;
        nhe++;
        const int endv = hf ? arc_ve(ci) : arc_vs(ci);
        if (endv == start_v) break;
        int nxt = -1;
        for (int j = 0; j < na && nxt < 0; j++) {
          const uint32_t aj = arcs[j].ids;
          if (arc_lo(aj) != 0 || usd[j]) continue;
          const int hj = ws.sign[arc_hi(aj)] < 0;
          if ((hj ? arc_vs(aj) : arc_ve(aj)) == endv) nxt = j;
        }
        if (nxt < 0) { st = LMM_NODE_HOLE; break; }
        cur = nxt;
      }
    }
    hoff[nh] = nhe;
    hs_st = st; hs_nh = nh; hs_nhe = nhe;
  }
  __syncthreads();
  if (hs_st) return hs_st;
  const int nh = hs_nh, nhe = hs_nhe;

  // ---- 7. slabs in a virtual slot of the overflow region ---------------------------------
  // virtual degree D: the smallest slab capacity K D + K0 that holds every count
  int D = ceil_div_pos(nv - SLAB_V_K0, SLAB_V_K);
  D = max(D, ceil_div_pos(na - SLAB_A_K0, SLAB_A_K));
  D = max(D, ceil_div_pos(nle - SLAB_L_K0, SLAB_L_K));
  D = max(D, ceil_div_pos(nh - SLAB_H_K0, SLAB_H_K));
  D = max(D, ceil_div_pos(nhe - SLAB_HE_K0, SLAB_HE_K));
  if (tid == 0) slot_sh = atomicAdd(&P.ctl[0], ((unsigned long long)D << 32) | 1ull);
  __syncthreads();
  const int64_t voff = (int64_t)(slot_sh >> 32), vn = (int64_t)(slot_sh & 0xffffffffull);
  if (voff + D > P.ovf_off || vn + 1 > P.ovf_n) {   // reserve exhausted: the host grows it and reruns
    if (tid == 0) atomicAdd(&P.ctl[2], 1ull);
    return 0;
  }
  const int64_t koff = P.S2 + voff, kn = P.N + vn;
  float4 *vslab = P.vert + slab_base(koff, kn, SLAB_V_K, SLAB_V_K0);
  uint32_t *vhi = P.vmask_hi + (slab_base(koff, kn, SLAB_V_K, SLAB_V_K0) - slab_base(P.S2, P.N, SLAB_V_K, SLAB_V_K0));
  for (int q = tid; q < nv; q += ST) {
    vslab[q] = make_float4(vx[q], vy[q], vz[q], __uint_as_float((uint32_t)vmask[q]));
    vhi[q] = (uint32_t)(vmask[q] >> 32);
  }
  ArcRec *aslab = P.arc + slab_base(koff, kn, SLAB_A_K, SLAB_A_K0);
  for (int i = tid; i < na; i += ST) aslab[i] = arcs[i];
  LoopRec *lslab = P.loop + slab_base(koff, kn, SLAB_L_K, SLAB_L_K0);
  for (int i = tid; i < nle; i += ST) lslab[i] = le[i];
  int2 *hslab = P.hole_hdr + slab_base(koff, kn, SLAB_H_K, SLAB_H_K0);
  for (int h = tid; h < nh; h += ST) hslab[h] = make_int2(hoff[h], hoff[h + 1] - hoff[h]);
  HoleEnt *heslab = P.hole_ent + slab_base(koff, kn, SLAB_HE_K, SLAB_HE_K0);
  for (int i = tid; i < nhe; i += ST) heslab[i] = he[i];
  for (int kk = tid; kk < d; kk += ST) P.loop_hdr[off + kk] = make_int2(lpos[kk + 1], lcnt[kk + 1]);
  if (tid == 0) {
    P.skey[n] = make_int2((int)koff, (int)kn);
    P.node_hdr[n] = make_int4(0 | (d << 8), nv | (na << 16), nh | (nle << 16), nhe);
  }
  return 0;
}

// a decided topology that is not a closed cell complex: re-decide at a coarser vertex resolution
__device__ __forceinline__ bool retry_status(int st) {
  return st == LMM_NODE_CHAIN || st == LMM_NODE_HOLE || st == LMM_NODE_UNREF || st == LMM_NODE_ANGLE || st == LMM_NODE_EMPTY;
}

__global__ void __launch_bounds__(ST, 1) k_spill(SpillParams P) {
  __shared__ SpillWS ws;
  for (int i = blockIdx.x; i < P.n_list; i += gridDim.x) {
    const int n = P.list[i];
    int64_t need = 0;
    int st = 0;
    for (int level = P.level[i]; level <= LMM_MAX_LEVEL; level++) {
      st = spill_node(P, ws, n, level, &need);
      __syncthreads();
      if (need > 0 || !retry_status(st)) break;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (need > 0) atomicMax(&P.ctl[1], (unsigned long long)need);
      else if (st != 0) {
        const int d = P.csr_off[n + 1] - P.csr_off[n];
        P.node_hdr[n] = make_int4(st | (d << 8), 0, 0, 0);
      }
    }
    if (st != 0 && need == 0) {
      const int off = P.csr_off[n], d = P.csr_off[n + 1] - off;
      for (int k = threadIdx.x; k < d; k += ST) P.loop_hdr[off + k] = make_int2(0, 0);
    }
    __syncthreads();
  }
}

// nodes left for the spill kernel: capacity refusals of the buckets and degrees 32..63 (from
// vertex resolution level 0), and bucketed nodes whose level-0 topology did not close (from level 1)
__global__ void k_spill_list(const int4 *node_hdr, int64_t N, int *list, int *level, unsigned long long *ctl) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int st = node_hdr[n].x & 0xff;
  const bool cap = st == LMM_NODE_JCAP || st == LMM_NODE_CCAP || st == LMM_NODE_ACAP || st == LMM_NODE_QCAP ||
                   st == LMM_NODE_SPILL;
  if (cap || retry_status(st)) {
    const int i = (int)atomicAdd(&ctl[3], 1ull);
    list[i] = (int)n;
    level[i] = cap ? 0 : 1;
  }
}

__global__ void k_skey_init(const int *csr_off, int64_t N, int2 *skey) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n < N) skey[n] = make_int2(csr_off[n], (int)n);
}

}  // namespace

int slab_key_init(lmm_ctx *c) {
  int rc;
  if ((rc = dev_alloc(c->skey, sizeof(int2) * (c->N + 1)))) return rc;
  if (c->N) {
    (c->n_launch++), k_skey_init<<<(unsigned)((c->N + 255) / 256), 256, 0, c->stream>>>((const int *)c->csr_off.p, c->N, (int2 *)c->skey.p);
    CUDA_TRY(cudaGetLastError());
  }
  return LMM_OK;
}

int spill_run(lmm_ctx *c) {
  const int64_t N = c->N;
  c->n_spill = 0;
  if (!N) return LMM_OK;
  int rc;
  if ((rc = dev_alloc(c->spill_ctl, sizeof(unsigned long long) * 8))) return rc;
  if ((rc = dev_alloc(c->spill_list, sizeof(int) * 2 * (N + 1)))) return rc;
  int *list = (int *)c->spill_list.p, *lvl = list + (N + 1);
  unsigned long long *ctl = (unsigned long long *)c->spill_ctl.p;
  CUDA_TRY(cudaMemsetAsync(ctl, 0, sizeof(unsigned long long) * 8, c->stream));
  (c->n_launch++), k_spill_list<<<(unsigned)((N + 255) / 256), 256, 0, c->stream>>>((const int4 *)c->node_hdr.p, N, list, lvl, ctl);
  CUDA_TRY(cudaGetLastError());
  if (!c->pinned_scalar) CUDA_TRY(cudaMallocHost((void **)&c->pinned_scalar, 64));
  unsigned long long *h = (unsigned long long *)(c->pinned_scalar + 4);   // 4 words
  CUDA_TRY(cudaMemcpyAsync(h, ctl, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const int64_t ns = (int64_t)h[3];
  c->n_spill = ns;
  if (ns == 0) return LMM_OK;
  if (c->spill_wsb < (1 << 20)) c->spill_wsb = 1 << 20;
  for (int attempt = 0; attempt < 24; attempt++) {
    const int grid = (int)(ns < c->n_sm ? ns : c->n_sm);
    if ((rc = dev_alloc(c->spill_ws, (size_t)c->spill_wsb * grid))) return rc;
    CUDA_TRY(cudaMemsetAsync(ctl, 0, sizeof(unsigned long long) * 3, c->stream));
    SpillParams P;
    P.node = (const float4 *)c->node.p;
    P.csr_off = (const int *)c->csr_off.p;
    P.csr_ent = (const int2 *)c->csr_ent.p;
    P.list = list;
    P.level = lvl;
    P.n_list = (int)ns;
    P.node_hdr = (int4 *)c->node_hdr.p;
    P.skey = (int2 *)c->skey.p;
    P.vert = (float4 *)c->vert.p;
    P.arc = (ArcRec *)c->arc.p;
    P.loop_hdr = (int2 *)c->loop_hdr.p;
    P.loop = (LoopRec *)c->loop.p;
    P.hole_hdr = (int2 *)c->hole_hdr.p;
    P.hole_ent = (HoleEnt *)c->hole_ent.p;
    P.vmask_hi = (uint32_t *)c->vmask_hi.p;
    P.S2 = 2 * c->S;
    P.N = N;
    P.ovf_off = c->ovf_off;
    P.ovf_n = c->ovf_n;
    P.ws = (unsigned char *)c->spill_ws.p;
    P.wsb = (int64_t)c->spill_wsb;
    P.ctl = ctl;
    (c->n_launch++), k_spill<<<grid, ST, 0, c->stream>>>(P);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(h, ctl, sizeof(unsigned long long) * 3, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    bool again = false;
    if ((int64_t)h[1] > c->spill_wsb) {        // a node needs a larger workspace
      c->spill_wsb = ((int64_t)h[1] + 4095) & ~(int64_t)4095;
      again = true;
    }
    if (h[2]) {                                 // the overflow slab reserve is exhausted
      const int64_t need_off = (int64_t)(h[0] >> 32), need_n = (int64_t)(h[0] & 0xffffffffull);
      if ((rc = slabs_alloc(c, need_off + need_off / 4 + 64, need_n + need_n / 4 + 16, true))) return rc;
      again = true;
    }
    if (!again) return LMM_OK;
  }
  return LMM_E_OOM;
}
