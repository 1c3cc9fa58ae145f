// metamesh.cu -- per-node meta-mesh kernel (Sec. 4.1, 4.3.1, Eq. 7-9).
//
// One lane group (8, 16 or 32 lanes by degree bucket: four, two or one node per warp) owns
// one lattice node; three part kernels (A: sides, junctions, vertex clusters; B: arcs;
// C: loops, holes, slab write) hand the node over through side records.  Lanes map to the
// node's struts for
// the per-side set-up, to (side, side, side) triples for the junction solve, to side
// pairs for the arc walk (Eq. 7 ellipse + interval tests, Eq. 8-9 read as
// the half-space tests at interval midpoints) and to struts for loop assembly; warp
// ballots compact the variable-length results in the deterministic order of
// DESIGN.md Sec. 4.  Nodes are scheduled through degree buckets (lattice.cu) so the
// warps of a CTA carry comparable work.
//
// COMPILED WITH -fmad=false: every binary32 operation below is rounded as written, so
// the topology decisions are bit-identical to the specification (and to the CPU
// oracle's, which evaluates the same operations).
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>

#include "lmm_internal.h"
#include "mm_node.cuh"

namespace cg = cooperative_groups;

#ifdef LMM_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[16];
extern "C" LMM_API int lmm_debug_phase_cycles(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles)) == cudaSuccess ? 0 : 2;
}
#endif

namespace {
using namespace mm;

// per-bucket workspace capacities <MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH> (degree 1-4, 5-8, 9-12, 13-16,
// 17-23, 24-31), sized for occupancy: a node that needs more (e.g. many coincident junctions)
// is meta-meshed by the spill kernel (spill.cu) -- the capacities never change a result
#define LMM_B00_ARGS 5, 24, 10, 14, 28, 10
#define LMM_B0_ARGS 9, 96, 18, 26, 52, 18
#define LMM_B1_ARGS 13, 96, 26, 38, 76, 26
#define LMM_B1b_ARGS 17, 96, 34, 50, 100, 34
#define LMM_B2_ARGS 24, 96, 48, 71, 142, 48
#define LMM_B3_ARGS 32, 128, 64, 95, 190, 64

struct MMParams {
  const float4 *node;
  const int *csr_off;
  const int2 *csr_ent;
  const int2 *ends;
  const int *node_list;
  int n_list;
  int4 *node_hdr;
  float4 *vert;
  ArcRec *arc;
  int2 *loop_hdr;
  LoopRec *loop;
  int2 *hole_hdr;
  HoleEnt *hole_ent;
  const uint32_t *tri3;   // lexicographic triples a | b << 8 | c << 16 of n sides at C(n,4)
  const uint32_t *pair2;  // lexicographic pairs a | b << 8 of n sides at C(n,3)
  float4 *side;    // [2S][5] side records between the parts (csr entry order)
  int4 *state;     // [N] status, clusters, vertices, arcs between the parts
};

// Per-warp shared-memory workspaces.  The meta-mesh of a node is built by three kernels
// (A: sides, junctions, vertex clusters; B: arcs; C: loops, holes, slab write) so that each
// kernel's code fits the instruction caches; every part keeps the sides and vertices.
template <int MAXS, int MAXV>
struct alignas(16) WSCore {
  // sides: 0 = nodal sphere, 1..d = incident struts in ascending strut id;
  // w4[k] = (w_k, e_k) of h_k(y) = w_k . y - e_k, one 16-byte load per side test
  float4 w4[MAXS];
  float ux[MAXS], uy[MAXS], uz[MAXS], s[MAXS], c[MAXS], L[MAXS];
  float asx[MAXS], asy[MAXS], asz[MAXS];
  float e1x[MAXS], e1y[MAXS], e1z[MAXS];
  float e2x[MAXS], e2y[MAXS], e2z[MAXS];
  int sign[MAXS];
  // vertices: clusters then seams
  float vx[MAXV], vy[MAXV], vz[MAXV];
  uint32_t vmask[MAXV];
};

// junction pre-test (part_a) for the buckets of at least this many sides (degree >= 13 by
// default: on the degree 9-12 octet nodes the pre-test costs more than it saves)
#ifndef LMM_PRE_MAXS
#define LMM_PRE_MAXS 17
#endif
#ifndef LMM_PRE_NN
#define LMM_PRE_NN 2   // nearest struts per side in the pre-test (1..3)
#endif
template <int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
struct alignas(16) WS_A : WSCore<MAXS, MAXV> {
  // side k as broadcast pairs for the two-root junction test: (wx,wx,wy,wy), (wz,wz,-e,-e)
  float4 wp[MAXS][2];
  float lim[MAXS];   // 0.45 L c of each strut side (SHORT limit); +inf for the sphere
  float4 jp[MAXJ];   // junction x, y, z; .w = vertex id once clustered (roots)
  uint32_t jabc[MAXJ];
  int jlab[MAXJ];
  // warp-per-node buckets: the roots that pass a pre-test against the triple's nearest sides,
  // queued (ring buffer) for the full side test in batches of 32 (see part_a)
  static constexpr int QA = MAXS >= LMM_PRE_MAXS ? 96 : 1;
  uint32_t nn[MAXS];     // the three struts nearest in direction to strut k (bytes 0, 1, 2)
  float4 jq[QA];         // queued root: x, y, z, solver tau
  uint32_t jqc[QA];      // its jabc code | sphere << 26 | SHORT << 27
};

#ifndef LMM_QL
#define LMM_QL 3
#endif
constexpr int QL = LMM_QL;   // arc-interval midpoints queued per lane and round (part B)

template <int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
struct alignas(16) WS_B : WSCore<MAXS, MAXV> {
  float4 wp[MAXS][2];   // side k as broadcast pairs (wx,wx,wy,wy), (wz,wz,-e,-e) for packed tests
  ArcRec arcs[MAXA];
  float atmid[MAXA];
  int adrop[MAXA];
  // active side pairs, each with the mask of the clusters holding both sides
  unsigned long long pmask[MAXS * (MAXS - 1) / 2];
  unsigned long long sclu[MAXS];   // per side: the clusters whose tie set holds it
  int plist[MAXS * (MAXS - 1) / 2];
  // queued interval midpoints
  float qx[32 * QL], qy[32 * QL], qz[32 * QL];
  int qt[32 * QL];
  uint32_t qm[32 * QL];
  int qok[32 * QL];
};

template <int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
struct alignas(16) WS_C : WSCore<MAXS, MAXV> {
  ArcRec arcs[MAXA];
  // loop entries of every (arc, side): phi start, span, forward flag
  float eps[2 * MAXA], edp[2 * MAXA];
  uint8_t efw[2 * MAXA];
  int lcnt[MAXS], lpos[MAXS], lfill[MAXS];
  int lslot[2 * MAXA];
  LoopRec le[MAXLE];
  int lfirst[MAXS], lcount[MAXS];
  int hoff[MAXH + 1];
  uint32_t he[MAXA];
};

template <int G> __device__ __forceinline__ int excl_scan(cg::thread_block_tile<G> &g, int v, int *total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < G; o <<= 1) {
    int y = g.shfl_up(x, o);
    if ((int)g.thread_rank() >= o) x += y;
  }
  *total = g.shfl(x, G - 1);
  return x - v;
}

// first lane (lowest rank) whose err != 0, its code; 0 if none
template <int G> __device__ __forceinline__ int first_err(cg::thread_block_tile<G> &g, int err) {
  unsigned m = g.ballot(err != 0);
  if (!m) return 0;
  return g.shfl(err, __ffs(m) - 1);
}



// vertices on one conic held per lane in part B (more: QCAP, the node goes to the spill kernel)
#ifndef LMM_MAXQ
#define LMM_MAXQ 16
#endif
#define MAXQ LMM_MAXQ
#define MAXLOOP 32

// side records between the parts: 5 float4 per CSR entry
template <int G, class WS>
__device__ void store_sides(cg::thread_block_tile<G> &g, const WS &ws, float4 *side, int off, int d) {
  #pragma unroll 1
  for (int idx = g.thread_rank(); idx < d; idx += G) {
    const int k = idx + 1;
    float4 *r = side + 5 * (int64_t)(off + idx);
    r[0] = ws.w4[k];
    r[1] = make_float4(ws.ux[k], ws.uy[k], ws.uz[k], ws.s[k]);
    r[2] = make_float4(ws.asx[k], ws.asy[k], ws.asz[k], ws.c[k]);
    r[3] = make_float4(ws.e1x[k], ws.e1y[k], ws.e1z[k], ws.L[k]);
    r[4] = make_float4(ws.e2x[k], ws.e2y[k], ws.e2z[k], __int_as_float(ws.sign[k]));
  }
}
template <int G, class WS>
__device__ void load_sides(cg::thread_block_tile<G> &g, WS &ws, const float4 *side, int off, int d) {
  if (g.thread_rank() == 0) ws.w4[0] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  #pragma unroll 1
  for (int idx = g.thread_rank(); idx < d; idx += G) {
    const int k = idx + 1;
    const float4 *r = side + 5 * (int64_t)(off + idx);
    const float4 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3], r4 = r[4];
    ws.w4[k] = r0;
    ws.ux[k] = r1.x; ws.uy[k] = r1.y; ws.uz[k] = r1.z; ws.s[k] = r1.w;
    ws.asx[k] = r2.x; ws.asy[k] = r2.y; ws.asz[k] = r2.z; ws.c[k] = r2.w;
    ws.e1x[k] = r3.x; ws.e1y[k] = r3.y; ws.e1z[k] = r3.z; ws.L[k] = r3.w;
    ws.e2x[k] = r4.x; ws.e2y[k] = r4.y; ws.e2z[k] = r4.z; ws.sign[k] = __float_as_int(r4.w);
  }
}
template <int G, class WS>
__device__ void store_verts(cg::thread_block_tile<G> &g, const WS &ws, float4 *vert, int q0, int q1) {
  #pragma unroll 1
  for (int q = q0 + g.thread_rank(); q < q1; q += G) vert[q] = make_float4(ws.vx[q], ws.vy[q], ws.vz[q], __uint_as_float(ws.vmask[q]));
}
template <int G, class WS>
__device__ void load_verts(cg::thread_block_tile<G> &g, WS &ws, const float4 *vert, int nv) {
  #pragma unroll 1
  for (int q = g.thread_rank(); q < nv; q += G) {
    const float4 v = vert[q];
    ws.vx[q] = v.x; ws.vy[q] = v.y; ws.vz[q] = v.z; ws.vmask[q] = __float_as_uint(v.w);
  }
}
template <int G>
__device__ void copy_arcs(cg::thread_block_tile<G> &g, ArcRec *dst, const ArcRec *src, int na) {
  const float4 *s4 = reinterpret_cast<const float4 *>(src);
  float4 *d4 = reinterpret_cast<float4 *>(dst);
  #pragma unroll 1
  for (int q = g.thread_rank(); q < na * 3; q += G) d4[q] = s4[q];
}

template <int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH, class WS>
__device__ void part_a(cg::thread_block_tile<G> &g, WS &ws, const MMParams &P, int n) {
  const int lane = g.thread_rank();
  const int off = P.csr_off[n];
  const int d = P.csr_off[n + 1] - off;
  const float4 on = P.node[n];
  Node<WS> nd{ws, d, on.w};
  const float R = on.w;
  const float delta = LMM_TOL_REL * R, dc = LMM_CTOL_REL * R;
  (void)dc;
  int status = 0;
#ifdef LMM_PHASE_TIMING
  long long ph_t = clock64();
#define PHASE_MARK(k)                                                    \
  do {                                                                   \
    long long ph_n = clock64();                                          \
    if (lane == 0) atomicAdd(&g_phase_cycles[(k) - 1], (unsigned long long)(ph_n - ph_t)); \
    ph_t = ph_n;                                                         \
  } while (0)
#else
#define PHASE_MARK(k) do { } while (0)
#endif
  // ---- 1. sides -------------------------------------------------------------------
  if (lane == 0) {
    ws.w4[0] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    ws.lim[0] = __int_as_float(0x7f800000);   // the sphere side never limits
  }
  int err = 0;
  #pragma unroll 1
  for (int k0 = 0; k0 < d; k0 += G) {
    int idx = k0 + lane;
    if (idx < d) {
      int k = idx + 1;
      int2 ent = P.csr_ent[off + idx];
      int far = ent.y & 0x7fffffff;
      int endbit = (unsigned)ent.y >> 31;
      if (!mm::setup_side(ws, k, on, P.node[far], endbit)) err = LMM_NODE_STRUT;
    }
  }
  if (g.any(err != 0)) status = LMM_NODE_STRUT;
  g.sync();

  int nj = 0, nc = 0, nv = 0, na = 0, nle = 0, nh = 0, nhe = 0;
  const int ns = d + 1;

  PHASE_MARK(1);
  // ---- 2. triple junctions, lexicographic (a<b<c), root-minor ---------------------
  // Warp-per-node buckets: a root's validity is an AND over the sides, so each root is first
  // tested against the (up to six) struts nearest in direction to its triple's sides -- its
  // likely violators -- and only the survivors, queued in (triple, root) order, take the full
  // side loop, 32 at a time.  Same operations on the same values: the decisions, the junction
  // order and the first error are those of the all-sides test below.
  constexpr bool PRE = G == 32 && WS::QA > 1;
  if constexpr (PRE) {
    if (status == 0 && d > 0) {
      #pragma unroll 1
      for (int k = 1 + lane; k <= d; k += G) {
        const f3 uk = nd.U(k);
        float b1 = -3.0f, b2 = -3.0f, b3 = -3.0f;
        int i1 = k, i2 = k, i3 = k;
        for (int m = 1; m <= d; m++) {
          if (m == k) continue;
          const float cm = f_dot(uk, nd.U(m));
          if (cm > b1) { b3 = b2; i3 = i2; b2 = b1; i2 = i1; b1 = cm; i1 = m; }
          else if (cm > b2) { b3 = b2; i3 = i2; b2 = cm; i2 = m; }
          else if (cm > b3) { b3 = cm; i3 = m; }
        }
        ws.nn[k] = (uint32_t)i1 | ((uint32_t)i2 << 8) | ((uint32_t)i3 << 16);
      }
      if (lane == 0) {
        ws.nn[0] = 0u;
        ws.wp[0][0] = make_float4(0.f, 0.f, 0.f, 0.f);
        ws.wp[0][1] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      g.sync();
      const int ntri = ns * (ns - 1) * (ns - 2) / 6;
      const uint32_t *t3 = P.tri3 + ns * (ns - 1) * (ns - 2) * (ns - 3) / 24;
      constexpr int QC = WS::QA;
      int qh = 0, nq = 0;   // queue head and length (warp-uniform)
      const unsigned lt = (1u << lane) - 1u;
      // the full side test of queued roots [qh, qh + cnt) (one per lane), appended in order
      auto drain_q = [&](int cnt) -> int {
        const int qi = qh + lane >= QC ? qh + lane - QC : qh + lane;
        bool v = false;
        uint32_t qc = 0u;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (lane < cnt) {
          q = ws.jq[qi];
          qc = ws.jqc[qi];
          const bool sphere = (qc >> 26) & 1u;
          const uint32_t excl = (1u << (qc & 0xff)) | (1u << ((qc >> 8) & 0xff)) | (1u << ((qc >> 16) & 0xff));
          const float tau = sphere ? 0.0f : q.w;
          const f3 y = F3(q.x, q.y, q.z);
          uint32_t viol = 0u, mb = 2u;
          for (int m = 1; m <= d; m++, mb <<= 1) viol |= (nd.hs(m, y) - tau > delta) ? mb : 0u;
          v = !(viol & ~excl);
        }
        const unsigned vm = g.ballot(v);
        const int pos = nj + __popc(vm & lt);
        int e = 0;
        if (v) e = pos >= MAXJ ? LMM_NODE_JCAP : (((qc >> 27) & 1u) ? LMM_NODE_SHORT : 0);
        const int fe = first_err<G>(g, e);
        if (fe) return fe;
        if (v) {
          ws.jp[pos] = make_float4(q.x, q.y, q.z, 0.0f);
          ws.jabc[pos] = qc & 0x03ffffffu;
        }
        nj += __popc(vm);
        qh = qh + cnt >= QC ? qh + cnt - QC : qh + cnt;
        nq -= cnt;
        return 0;
      };
      #pragma unroll 1
      for (int base = 0; base < ntri && status == 0; base += G) {
        const int t = base + lane;
        const uint32_t code = __ldg(&t3[t < ntri ? t : ntri - 1]);
        const int a = code & 0xff, b = (code >> 8) & 0xff, c = code >> 16;
        f3 y[2];
        float tau[2];
        const bool solved = nd.junction_bf(a, b, c, y, tau) && t < ntri;
        const uint32_t excl = (1u << a) | (1u << b) | (1u << c);
        const bool sphere = a == 0;
        bool v0 = solved && (sphere || !(tau[0] < -delta)), v1 = solved && (sphere || !(tau[1] < -delta));
        {   // pre-test: the nearest struts of a, b, c, both roots in packed f32x2 operations
          const float2 Yx = make_float2(y[0].x, y[1].x), Yy = make_float2(y[0].y, y[1].y), Yz = make_float2(y[0].z, y[1].z);
          const float2 nT = sphere ? make_float2(0.0f, 0.0f) : make_float2(-tau[0], -tau[1]);
          const uint32_t la = ws.nn[a], lb = ws.nn[b], lc = ws.nn[c];
          uint32_t w0 = 0u, w1 = 0u;
          #pragma unroll
          for (int r = 0; r < 3 * LMM_PRE_NN; r++) {
            const uint32_t lw = r < LMM_PRE_NN ? la : (r < 2 * LMM_PRE_NN ? lb : lc);
            const int m = (lw >> (8 * (r % LMM_PRE_NN))) & 0xff;
            const float2 h = side_h2(ws.wp[m][0], ws.wp[m][1], Yx, Yy, Yz, nT);
            w0 |= h.x > delta ? 1u << m : 0u;
            w1 |= h.y > delta ? 1u << m : 0u;
          }
          v0 = v0 && !(w0 & ~excl);
          v1 = v1 && !(w1 & ~excl);
        }
        const unsigned m0 = g.ballot(v0), m1 = g.ballot(v1);
        if (m0 | m1) {
          const float lm = fminf(fminf(ws.lim[a], ws.lim[b]), ws.lim[c]);
          int qp = qh + nq + __popc(m0 & lt) + __popc(m1 & lt);
          qp = qp >= QC ? qp - QC : qp;
          const uint32_t cf = code | (sphere ? (1u << 26) : 0u);
          if (v0) {
            ws.jq[qp] = make_float4(y[0].x, y[0].y, y[0].z, tau[0]);
            ws.jqc[qp] = cf | (fabsf(tau[0]) <= delta ? (1u << 25) : 0u) | (tau[0] > lm ? (1u << 27) : 0u);
          }
          if (v1) {
            const int q1 = qp + (v0 ? 1 : 0) >= QC ? qp + (v0 ? 1 : 0) - QC : qp + (v0 ? 1 : 0);
            ws.jq[q1] = make_float4(y[1].x, y[1].y, y[1].z, tau[1]);
            ws.jqc[q1] = cf | (1u << 24) | (fabsf(tau[1]) <= delta ? (1u << 25) : 0u) | (tau[1] > lm ? (1u << 27) : 0u);
          }
          nq += __popc(m0) + __popc(m1);
          g.sync();
          while (nq >= G && status == 0) status = drain_q(G);
        }
      }
      if (status == 0 && nq > 0) status = drain_q(nq);
    }
  }
  if (!PRE && status == 0 && d > 0) {
    const int ntri = ns * (ns - 1) * (ns - 2) / 6;
    const uint32_t *t3 = P.tri3 + ns * (ns - 1) * (ns - 2) * (ns - 3) / 24;   // triples of ns sides
    #pragma unroll 1
    for (int base = 0; base < ntri; base += G) {
      int t = base + lane;
      bool v0 = false, v1 = false;
      int a = 0, b = 0, c = 0;
      f3 y[2];
      float tau[2];
      bool sh0 = false, sh1 = false;
      {
        // every lane of the group runs the same straight-line solve and side loop
        const uint32_t code = __ldg(&t3[t < ntri ? t : ntri - 1]);
        a = code & 0xff; b = (code >> 8) & 0xff; c = code >> 16;
        const bool solved = nd.junction_bf(a, b, c, y, tau) && t < ntri;
        const uint32_t excl = (1u << a) | (1u << b) | (1u << c);
        v0 = v1 = solved;
        nd.valid_junction_pair(a == 0, excl, y[0], tau[0], y[1], tau[1], delta, &v0, &v1);
        // strut too short: tau above 0.45 L c of any strut side of the triple
        const float lm = fminf(fminf(ws.lim[a], ws.lim[b]), ws.lim[c]);
        sh0 = v0 && tau[0] > lm;
        sh1 = v1 && tau[1] > lm;
      }
      unsigned m0 = g.ballot(v0), m1 = g.ballot(v1);
      unsigned lt = (1u << lane) - 1u;
      int pos = nj + __popc(m0 & lt) + __popc(m1 & lt);
      int p0 = pos, p1 = pos + (v0 ? 1 : 0);
      int e = 0;
      if (v0) e = p0 >= MAXJ ? LMM_NODE_JCAP : (sh0 ? LMM_NODE_SHORT : 0);
      if (!e && v1) e = p1 >= MAXJ ? LMM_NODE_JCAP : (sh1 ? LMM_NODE_SHORT : 0);
      int fe = first_err<G>(g, e);
      if (fe) { status = fe; break; }
      uint32_t code = (uint32_t)a | ((uint32_t)b << 8) | ((uint32_t)c << 16);
      if (v0) {
        ws.jp[p0] = make_float4(y[0].x, y[0].y, y[0].z, 0.0f);
        ws.jabc[p0] = code | (fabsf(tau[0]) <= delta ? (1u << 25) : 0u);
      }
      if (v1) {
        ws.jp[p1] = make_float4(y[1].x, y[1].y, y[1].z, 0.0f);
        ws.jabc[p1] = code | (1u << 24) | (fabsf(tau[1]) <= delta ? (1u << 25) : 0u);
      }
      nj += __popc(m0) + __popc(m1);
    }
  }
  g.sync();

  PHASE_MARK(2);
  // ---- 3. clustering: connected components of "junctions within delta_c" -----------
  // (label = lowest junction index of the component).  Up to MJ junctions: one pass builds
  // each junction's proximity mask (coordinates broadcast from shared memory), the masks
  // are closed under union in place (monotone; clusters are small, so 1-2 sweeps), and the
  // component minimum is the lowest set bit.  More junctions: label propagation.
  if (status == 0 && nj > 0) {
    constexpr int MJW = (int)(sizeof(ws.wp) / sizeof(unsigned long long));   // masks fit in ws.wp
    constexpr int MJ = MJW >= 64 ? 64 : MJW;
    unsigned long long *msk = reinterpret_cast<unsigned long long *>(&ws.wp[0][0]);   // dead after step 2
    const bool masks = nj <= MJ;
    if (masks) {
      #pragma unroll 1
      for (int cj = 0; cj < nj; cj += G) {
        const int j = cj + lane;
        const float4 pj = j < nj ? ws.jp[j] : make_float4(0.f, 0.f, 0.f, 0.f);
        // max-norm distance (exact: max and abs do not round); bits shifted in from the top
        // junction down, as two 32-bit halves
        auto near = [&](int k) -> uint32_t {
          const float4 pk = ws.jp[k];
          const float dm = fmaxf(fmaxf(fabsf(pj.x - pk.x), fabsf(pj.y - pk.y)), fabsf(pj.z - pk.z));
          return dm <= dc ? 1u : 0u;
        };
        uint32_t hi = 0u, lo = 0u;
        #pragma unroll 4
        for (int k = nj - 1; k >= 32; k--) hi = (hi << 1) | near(k);
        #pragma unroll 4
        for (int k = (nj < 32 ? nj : 32) - 1; k >= 0; k--) lo = (lo << 1) | near(k);
        if (j < nj) msk[j] = ((unsigned long long)hi << 32) | lo;
      }
      g.sync();
      for (;;) {
        bool changed = false;
        #pragma unroll 1
        for (int j = lane; j < nj; j += G) {
          const unsigned long long R = msk[j];
          unsigned long long nr = R, bits = R & ~(1ull << j);
          while (bits) {
            nr |= msk[__ffsll((long long)bits) - 1];
            bits &= bits - 1;
          }
          if (nr != R) { msk[j] = nr; changed = true; }
        }
        g.sync();
        if (!g.any(changed)) break;
      }
      #pragma unroll 1
      for (int j = lane; j < nj; j += G) ws.jlab[j] = __ffsll((long long)msk[j]) - 1;
    } else {
      #pragma unroll 1
      for (int j = lane; j < nj; j += G) ws.jlab[j] = j;
      g.sync();
      for (;;) {
        bool changed = false;
        #pragma unroll 1
        for (int cj = 0; cj < nj; cj += G) {
          const int j = cj + lane;
          const bool vj = j < nj;
          const float4 pj = vj ? ws.jp[j] : make_float4(0.f, 0.f, 0.f, 0.f);
          int lj = vj ? ws.jlab[j] : 0x7fffffff;
          #pragma unroll 1
          for (int k = 0; k < nj; k++) {
            const float4 pk = ws.jp[k];
            const int lk = ws.jlab[k];
            if (lk < lj && fabsf(pj.x - pk.x) <= dc && fabsf(pj.y - pk.y) <= dc && fabsf(pj.z - pk.z) <= dc) lj = lk;
          }
          g.sync();
          if (vj && lj != ws.jlab[j]) { ws.jlab[j] = lj; changed = true; }
          g.sync();
        }
        if (!g.any(changed)) break;
      }
    }
    g.sync();
    // component roots in index order -> vertex ids (kept in the root's .w)
    #pragma unroll 1
    for (int base = 0; base < nj; base += G) {
      int j = base + lane;
      bool root = j < nj && ws.jlab[j] == j;
      unsigned rm = g.ballot(root);
      int id = nc + __popc(rm & ((1u << lane) - 1u));
      if (root && id < MAXV) {
        const float4 q = ws.jp[j];
        ws.jp[j].w = __int_as_float(id);
        ws.vx[id] = q.x; ws.vy[id] = q.y; ws.vz[id] = q.z; ws.vmask[id] = 0u;
      }
      nc += __popc(rm);
    }
    if (nc > MAXV) status = LMM_NODE_CCAP;
    g.sync();
    if (status == 0) {
      #pragma unroll 1
      for (int j = lane; j < nj; j += G) {
        uint32_t code = ws.jabc[j];
        uint32_t bits = (1u << (code & 0xff)) | (1u << ((code >> 8) & 0xff)) | (1u << ((code >> 16) & 0xff));
        if (code & (1u << 25)) bits |= 1u;   // strut junction at tangent length ~0: on the sphere
        atomicOr(&ws.vmask[__float_as_int(ws.jp[ws.jlab[j]].w)], bits);
      }
    }
  }
  nv = nc;
  g.sync();

  PHASE_MARK(3);
  // vertices to their slab, sides to the side records, state for part B
  if (status == 0 && nc > slab_cap(d, SLAB_V_K, SLAB_V_K0)) status = LMM_NODE_ACAP;
  if (status == 0) {
    store_sides<G>(g, ws, P.side, off, d);
    store_verts<G>(g, ws, P.vert + slab_base(off, n, SLAB_V_K, SLAB_V_K0), 0, nc);
  }
  if (lane == 0) P.state[n] = make_int4(status, nc, nc, 0);
  (void)nj; (void)na; (void)nle; (void)nh; (void)nhe;
  g.sync();
}

template <int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH, class WS>
__device__ void part_b(cg::thread_block_tile<G> &g, WS &ws, const MMParams &P, int n) {
  const int lane = g.thread_rank();
  const int off = P.csr_off[n];
  const int d = P.csr_off[n + 1] - off;
  const float4 on = P.node[n];
  Node<WS> nd{ws, d, on.w};
  const float R = on.w;
  const float delta = LMM_TOL_REL * R, dc = LMM_CTOL_REL * R;
  (void)dc;
  const int4 st = P.state[n];
  int status = st.x;
  if (status != 0) return;
  const int nc = st.y;
  int nv = st.z, na = 0;
  const int ns = d + 1;
  float4 *vslab = P.vert + slab_base(off, n, SLAB_V_K, SLAB_V_K0);
  load_sides<G>(g, ws, P.side, off, d);
  load_verts<G>(g, ws, vslab, nv);
  g.sync();
  #pragma unroll 1
  for (int k = 1 + lane; k <= d; k += G) {
    const float4 q = ws.w4[k];
    ws.wp[k][0] = make_float4(q.x, q.x, q.y, q.y);
    ws.wp[k][1] = make_float4(q.z, q.z, -q.w, -q.w);
  }
  g.sync();
#ifdef LMM_PHASE_TIMING
  long long ph_t = clock64();
#define PHASE_MARK(k)                                                    \
  do {                                                                   \
    long long ph_n = clock64();                                          \
    if (lane == 0) atomicAdd(&g_phase_cycles[(k) - 1], (unsigned long long)(ph_n - ph_t)); \
    ph_t = ph_n;                                                         \
  } while (0)
#else
#define PHASE_MARK(k) do { } while (0)
#endif
  // ---- 4. arcs: conics walked through their vertices, incidence-driven --------------
  // Each side pair collects the clusters whose tie set holds both sides (a bit mask);
  // the pairs with vertices -- plus pairs of sides that appear in no vertex (only these
  // can carry a closed arc) -- are compacted in lexicographic order and walked densely.
  if (status == 0 && d > 0) {
    const int npair = ns * (ns - 1) / 2;
    uint32_t um = 0;
    #pragma unroll 1
    for (int q = lane; q < nc; q += G) um |= ws.vmask[q];
    um = cg::reduce(g, um, cg::bit_or<uint32_t>());
    // one lane per side pair: the clusters whose tie set holds both sides (nc <= MAXV <= 64),
    // the intersection of the two sides' cluster sets
    #pragma unroll 1
    for (int k = lane; k < ns; k += G) {
      unsigned long long m = 0ull;
      for (int q = 0; q < nc; q++) m |= (unsigned long long)((ws.vmask[q] >> k) & 1u) << q;
      ws.sclu[k] = m;
    }
    g.sync();
    int nact = 0;
    {
      #pragma unroll 1
      for (int base = 0; base < npair; base += G) {
        const int p = base + lane;
        bool act = false;
        unsigned long long cm = 0ull;
        if (p < npair) {
          const uint32_t pc = __ldg(&P.pair2[ns * (ns - 1) * (ns - 2) / 6 + p]);
          const int a = pc & 0xff, b = pc >> 8;
          const uint32_t pb = (1u << a) | (1u << b);
          cm = ws.sclu[a] & ws.sclu[b];
          const uint32_t strut_bits = a == 0 ? (1u << b) : pb;
          act = cm != 0ull || (um & strut_bits) == 0;
        }
        const unsigned am = g.ballot(act);
        if (act) {
          const int k = nact + __popc(am & ((1u << lane) - 1u));
          ws.plist[k] = p;
          ws.pmask[k] = cm;
        }
        nact += __popc(am);
      }
      g.sync();
      PHASE_MARK(9);
      float *qx = ws.qx, *qy = ws.qy, *qz = ws.qz;
      int *qt = ws.qt;          // tangent length at the midpoint, float bits
      uint32_t *qm = ws.qm;     // side mask | sphere-point flag << 31
      int *qok = ws.qok;
      #pragma unroll 1
      for (int base = 0; base < nact; base += G) {
        int k = base + lane;
        int e = 0, cnt = 0, closed = 0, nint = 0;
        int a = 0, b = 0;
        f3 o = F3(0.f, 0.f, 0.f), av = o, bv = o;
        int vsv[MAXQ], vev[MAXQ];
        float t0v[MAXQ], dtv[MAXQ], tmv[MAXQ];
        bool okv[MAXQ];
        int p = 0, nq = 0;
        unsigned long long cmk = 0ull;
        bool conic_ok = true;
        if (k < nact) {
          p = ws.plist[k];
          const uint32_t pc = __ldg(&P.pair2[ns * (ns - 1) * (ns - 2) / 6 + p]);
          a = pc & 0xff; b = pc >> 8;
          cmk = ws.pmask[k];
          nq = __popcll(cmk);
          if (a == 0) nd.circle(b, &o, &av, &bv);
          else conic_ok = nd.ellipse(a, b, &o, &av, &bv);
          if (!conic_ok) {
            if (nq > 0) e = LMM_NODE_CONIC;
          } else if (nq > MAXQ) {
            e = LMM_NODE_QCAP;
          } else nint = nq == 0 ? 1 : nq;
        }
        int qtot;
        const int qbase = excl_scan<G>(g, nint < QL ? nint : QL, &qtot);
        if (nint > 0) {
          const uint32_t pm = (1u << a) | (1u << b);
          int Q[MAXQ];
          float tq[MAXQ], us[MAXQ], uc[MAXQ];
          unsigned long long cmr = cmk;
          for (int i = 0; i < nq; i++, cmr &= cmr - 1) {
            const int q = __ffsll((long long)cmr) - 1;
            float su, sc;
            float t = conic_t(o, av, bv, nd.V(q), &su, &sc);
            int j = i;   // insertion by (t, cluster index): order-independent
            while (j > 0 && (t < tq[j - 1] || (t == tq[j - 1] && q < Q[j - 1]))) {
              Q[j] = Q[j - 1]; tq[j] = tq[j - 1]; us[j] = us[j - 1]; uc[j] = uc[j - 1];
              j--;
            }
            Q[j] = q; tq[j] = t; us[j] = su; uc[j] = sc;
          }
          for (int i = 0; i < nint; i++) {
            float ms, mc, t0, dt;
            int vs, ve;
            if (nq == 0) { ms = 0.0f; mc = 1.0f; t0 = 0.0f; dt = LMM_TWO_PI_F; vs = ve = -1; }
            else if (nq == 1) { ms = -us[0]; mc = -uc[0]; t0 = tq[0]; dt = LMM_TWO_PI_F; vs = ve = Q[0]; }
            else {
              int j = i + 1 == nq ? 0 : i + 1;
              dt = j == 0 ? (tq[0] + LMM_TWO_PI_F) - tq[nq - 1] : tq[j] - tq[i];
              if (!(dt > 0.0f)) { e = LMM_NODE_CHAIN; break; }
              float sx = us[i] + us[j], sc = uc[i] + uc[j];
              float l2 = sx * sx + sc * sc;
              if (l2 > 1e-6f) {
                float l = sqrtf(l2);
                ms = sx / l; mc = sc / l;
                if (dt > LMM_PI_F) { ms = -ms; mc = -mc; }
              } else { ms = uc[i]; mc = -us[i]; }
              t0 = tq[i]; vs = Q[i]; ve = Q[j];
            }
            f3 y = F3((o.x + av.x * ms) + bv.x * mc, (o.y + av.y * ms) + bv.y * mc, (o.z + av.z * ms) + bv.z * mc);
            float tmid = a == 0 ? 0.0f : nd.h(a, y);
            vsv[i] = vs; vev[i] = ve; t0v[i] = t0; dtv[i] = dt; tmv[i] = tmid;
            if (i < QL) {
              const int qi = qbase + i;
              qx[qi] = y.x; qy[qi] = y.y; qz[qi] = y.z; qt[qi] = __float_as_int(tmid);
              qm[qi] = pm | (a == 0 ? 0x80000000u : 0u);
            } else {
              okv[i] = a == 0 ? nd.valid_sphere_pt(pm, y, delta) : nd.valid_strut_pt(pm, y, tmid, delta);
            }
          }
        }
        g.sync();
        PHASE_MARK(10);
        // (2) queued midpoints: end-circle points strictly exposed (h_m - 0 > -delta
        // rejects, as valid_sphere_pt), strut points within the tolerance (valid_strut_pt)
        // two midpoints per lane in packed f32x2 operations: each lane of the pair rounds like
        // the scalar hs(m, y) - tau (h - e as h + (-e), h - tau as h + (-tau))
        for (int qi = lane; qi < qtot; qi += 2 * G) {
          const int qj = qi + G < qtot ? qi + G : qi;
          const uint32_t m0 = qm[qi], m1 = qm[qj];
          const bool s0 = m0 >> 31, s1 = m1 >> 31;
          const float t0 = __int_as_float(qt[qi]), t1 = __int_as_float(qt[qj]);
          const float th0 = s0 ? -delta : delta, th1 = s1 ? -delta : delta;
          bool ok0 = s0 || !(t0 < -delta), ok1 = s1 || !(t1 < -delta);
          const float2 Yx = make_float2(qx[qi], qx[qj]), Yy = make_float2(qy[qi], qy[qj]), Yz = make_float2(qz[qi], qz[qj]);
          const float2 nT = make_float2(-t0, -t1);
          uint32_t v0 = 0u, v1 = 0u, mb = 2u;   // sides violated at each midpoint (bit mm)
          for (int mm = 1; mm <= d; mm++, mb <<= 1) {
            const float4 p0 = ws.wp[mm][0], p1 = ws.wp[mm][1];
            const float2 h = side_h2(p0, p1, Yx, Yy, Yz, nT);
            v0 |= h.x > th0 ? mb : 0u;
            v1 |= h.y > th1 ? mb : 0u;
          }
          ok0 = ok0 && !(v0 & ~m0 & 0x7fffffffu);
          ok1 = ok1 && !(v1 & ~m1 & 0x7fffffffu);
          qok[qi] = ok0;
          if (qj != qi) qok[qj] = ok1;
        }
        g.sync();
        PHASE_MARK(11);
        // (3) valid intervals become arcs
        for (int i = 0; i < nint && !e; i++) {
          const bool ok = i < QL ? qok[qbase + i] != 0 : okv[i];
          if (!ok) continue;
          if (cnt != i) { vsv[cnt] = vsv[i]; vev[cnt] = vev[i]; t0v[cnt] = t0v[i]; dtv[cnt] = dtv[i]; tmv[cnt] = tmv[i]; }
          if (vsv[cnt] < 0) closed = 1;
          cnt++;
        }
        int tot, ctot;
        int pos = na + excl_scan<G>(g, e ? 0 : cnt, &tot);
        int spos = nv + excl_scan<G>(g, e ? 0 : closed, &ctot);
        if (!e && cnt > 0 && pos + cnt > MAXA) e = LMM_NODE_ACAP;
        if (!e && closed && spos >= MAXV) e = LMM_NODE_ACAP;
        int fe = first_err<G>(g, e);
        if (fe) { status = fe; break; }
        for (int i = 0; i < cnt; i++) {
          ArcRec &A = ws.arcs[pos + i];
          int vs = vsv[i], ve = vev[i];
          if (vs < 0) {
            ws.vx[spos] = o.x + bv.x; ws.vy[spos] = o.y + bv.y; ws.vz[spos] = o.z + bv.z;
            ws.vmask[spos] = (1u << a) | (1u << b);
            vs = ve = spos;
          }
          A.ids = arc_ids(a, b, vs, ve);
          A.t0 = t0v[i]; A.dt = dtv[i];
          ws.atmid[pos + i] = tmv[i];
          A.ox = o.x; A.oy = o.y; A.oz = o.z;
          A.ax = av.x; A.ay = av.y; A.az = av.z;
          A.bx = bv.x; A.by = bv.y; A.bz = bv.z;
        }
        na += tot;
        nv += ctot;
        PHASE_MARK(12);
      }
    }
  }
  g.sync();

  PHASE_MARK(4);
  // ambiguous strut-strut arcs running under a strictly exposed hole lune are dropped
  // (R10): midpoint tangent length < delta and both end circles join its ends
  if (status == 0 && na > 0) {
    #pragma unroll 1
    for (int i = lane; i < na; i += G) {
      uint32_t ids = ws.arcs[i].ids;
      int lo = arc_lo(ids), hi = arc_hi(ids), vs = arc_vs(ids), ve = arc_ve(ids);
      int drop = 0;
      if (lo > 0 && vs != ve && ws.atmid[i] < delta) {
        int ca = 0, cb = 0;
        for (int j = 0; j < na; j++) {
          uint32_t jd = ws.arcs[j].ids;
          if (arc_lo(jd) != 0) continue;
          int js = arc_vs(jd), je = arc_ve(jd), jh = arc_hi(jd);
          if (!((js == vs && je == ve) || (js == ve && je == vs))) continue;
          if (jh == lo) ca = 1;
          if (jh == hi) cb = 1;
        }
        drop = ca && cb;
      }
      ws.adrop[i] = drop;
    }
    g.sync();
    int w = 0;
    #pragma unroll 1
    for (int base = 0; base < na; base += G) {
      int i = base + lane;
      bool keep = i < na && !ws.adrop[i];
      ArcRec rec;
      if (keep) rec = ws.arcs[i];
      unsigned km = g.ballot(keep);
      g.sync();
      if (keep) ws.arcs[w + __popc(km & ((1u << lane) - 1u))] = rec;
      w += __popc(km);
      g.sync();
    }
    na = w;
  }
  g.sync();

  // every junction vertex must carry an arc (vertex ids < MAXV <= 64: one bit each)
  if (status == 0) {
    unsigned long long used = 0ull;
    #pragma unroll 1
    for (int i = lane; i < na; i += G) {
      const uint32_t ids = ws.arcs[i].ids;
      used |= (1ull << arc_vs(ids)) | (1ull << arc_ve(ids));
    }
    used = cg::reduce(g, used, cg::bit_or<unsigned long long>());
    const unsigned long long need = nc >= 64 ? ~0ull : (1ull << nc) - 1ull;
    if ((used & need) != need) status = LMM_NODE_UNREF;
  }

  // seam vertices and arcs to their slabs, state for part C
  if (status == 0 && (nv > slab_cap(d, SLAB_V_K, SLAB_V_K0) || na > slab_cap(d, SLAB_A_K, SLAB_A_K0)))
    status = LMM_NODE_ACAP;
  if (status == 0) {
    store_verts<G>(g, ws, vslab, nc, nv);
    copy_arcs<G>(g, P.arc + slab_base(off, n, SLAB_A_K, SLAB_A_K0), ws.arcs, na);
  }
  if (lane == 0) P.state[n] = make_int4(status, nc, nv, na);
  g.sync();
}

template <int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH, class WS>
__device__ void part_c(cg::thread_block_tile<G> &g, WS &ws, const MMParams &P, int n) {
  const int lane = g.thread_rank();
  const int off = P.csr_off[n];
  const int d = P.csr_off[n + 1] - off;
  const float4 on = P.node[n];
  Node<WS> nd{ws, d, on.w};
  const float R = on.w;
  const float dc = LMM_CTOL_REL * R;
  (void)dc;
  const int4 st = P.state[n];
  int status = st.x;
  int nv = status == 0 ? st.z : 0, na = status == 0 ? st.w : 0, nle = 0, nh = 0, nhe = 0;
  if (status == 0) {
    load_sides<G>(g, ws, P.side, off, d);
    load_verts<G>(g, ws, P.vert + slab_base(off, n, SLAB_V_K, SLAB_V_K0), nv);
    copy_arcs<G>(g, ws.arcs, P.arc + slab_base(off, n, SLAB_A_K, SLAB_A_K0), na);
  }
  g.sync();
#ifdef LMM_PHASE_TIMING
  long long ph_t = clock64();
#define PHASE_MARK(k)                                                    \
  do {                                                                   \
    long long ph_n = clock64();                                          \
    if (lane == 0) atomicAdd(&g_phase_cycles[(k) - 1], (unsigned long long)(ph_n - ph_t)); \
    ph_t = ph_n;                                                         \
  } while (0)
#else
#define PHASE_MARK(k) do { } while (0)
#endif
  // ---- 5. arc loops per strut end (ordered by angle around the strut axis) -----------
  if (status == 0 && d > 0) {
    // 5a: loop-entry data of every (arc, strut side), lanes over arcs
    #pragma unroll 1
    for (int i = lane; i < na; i += G) {
      const ArcRec &A = ws.arcs[i];
      const int lo = arc_lo(A.ids), hi = arc_hi(A.ids);
      const int avs = arc_vs(A.ids), ave = arc_ve(A.ids);
      for (int x = 0; x < 2; x++) {
        int k = x ? hi : lo;
        if (k == 0) continue;
        f3 as = nd.AS(k), e1 = nd.E1(k), e2 = nd.E2(k);
        int fwd = f_dot(f_cross(F3(A.ax, A.ay, A.az), F3(A.bx, A.by, A.bz)), as) < 0.0f;
        int vs = fwd ? avs : ave, ve = fwd ? ave : avs;
        f3 Ps = nd.V(vs);
        float ps = atan2p(f_dot(Ps, e2), f_dot(Ps, e1));
        if (ps < 0.0f) ps += LMM_TWO_PI_F;
        float dph;
        if (vs == ve) dph = LMM_TWO_PI_F;
        else {
          f3 Pe = nd.V(ve);
          float pe = atan2p(f_dot(Pe, e2), f_dot(Pe, e1));
          if (pe < 0.0f) pe += LMM_TWO_PI_F;
          dph = pe - ps;
          if (dph <= 0.0f) dph += LMM_TWO_PI_F;
        }
        ws.eps[2 * i + x] = ps;
        ws.edp[2 * i + x] = dph;
        ws.efw[2 * i + x] = (uint8_t)fwd;
      }
    }
    g.sync();
    // 5b: counting sort of the (arc, side) entries by strut side (shared atomics), then each
    // strut orders its few entries by (phi, arc index) and checks the chain
    #pragma unroll 1
    for (int k = lane; k <= d; k += G) { ws.lcnt[k] = 0; ws.lfill[k] = 0; }
    g.sync();
    #pragma unroll 1
    for (int i = lane; i < na; i += G) {
      uint32_t ids = ws.arcs[i].ids;
      int lo = arc_lo(ids), hi = arc_hi(ids);
      if (lo) atomicAdd(&ws.lcnt[lo], 1);
      atomicAdd(&ws.lcnt[hi], 1);
    }
    g.sync();
    {
      int run = 0;
      #pragma unroll 1
      for (int k0 = 0; k0 <= d; k0 += G) {
        int k = k0 + lane;
        int v = k <= d ? ws.lcnt[k] : 0, tot;
        int ex = excl_scan<G>(g, v, &tot);
        if (k <= d) ws.lpos[k] = run + ex;
        run += tot;
      }
    }
    g.sync();
    #pragma unroll 1
    for (int i = lane; i < na; i += G) {
      uint32_t ids = ws.arcs[i].ids;
      int lo = arc_lo(ids), hi = arc_hi(ids);
      if (lo) ws.lslot[ws.lpos[lo] + atomicAdd(&ws.lfill[lo], 1)] = 2 * i;
      ws.lslot[ws.lpos[hi] + atomicAdd(&ws.lfill[hi], 1)] = 2 * i + 1;
    }
    g.sync();
    #pragma unroll 1
    for (int k0 = 0; k0 < d; k0 += G) {
      int k = k0 + lane + 1;
      int e = 0, cnt = 0;
      int slot[MAXLOOP];
      if (k <= d) {
        const int n = ws.lcnt[k], p0 = ws.lpos[k];
        if (n > MAXLOOP) e = LMM_NODE_ACAP;
        else
          for (int t = 0; t < n; t++) {
            int sl = ws.lslot[p0 + t];
            float ps = ws.eps[sl];
            int j = cnt;   // insertion by (phi, arc index)
            while (j > 0 && (ps < ws.eps[slot[j - 1]] || (ps == ws.eps[slot[j - 1]] && sl < slot[j - 1]))) {
              slot[j] = slot[j - 1];
              j--;
            }
            slot[j] = sl;
            cnt++;
          }
        if (!e && cnt == 0) e = LMM_NODE_EMPTY;
        if (!e) {
          float sum = 0.0f;
          for (int i = 0; i < cnt; i++) {
            int sx = slot[i], sy = slot[(i + 1) % cnt];
            const uint32_t X = ws.arcs[sx >> 1].ids, Y = ws.arcs[sy >> 1].ids;
            int xe = ws.efw[sx] ? arc_ve(X) : arc_vs(X);
            int ys = ws.efw[sy] ? arc_vs(Y) : arc_ve(Y);
            if (xe != ys) { e = LMM_NODE_CHAIN; break; }
            sum += ws.edp[sx];
          }
          if (!e && fabsf(sum - LMM_TWO_PI_F) > 1e-3f) e = LMM_NODE_ANGLE;
        }
      }
      int tot;
      int pos = nle + excl_scan<G>(g, e ? 0 : cnt, &tot);
      if (!e && cnt > 0 && pos + cnt > MAXLE) e = LMM_NODE_ACAP;
      int fe = first_err<G>(g, e);
      if (fe) { status = fe; break; }
      if (k <= d) {
        ws.lfirst[k] = pos;
        ws.lcount[k] = cnt;
        float ph = cnt ? ws.eps[slot[0]] : 0.0f;
        for (int i = 0; i < cnt; i++) {
          if (i > 0) ph = ph + ws.edp[slot[i - 1]];
          LoopRec &L = ws.le[pos + i];
          const uint32_t aid = ws.arcs[slot[i] >> 1].ids;
          L.arc_fwd = (uint32_t)(slot[i] >> 1) | ((uint32_t)ws.efw[slot[i]] << 16);
          L.phs = ph;
          L.dph = ws.edp[slot[i]];
          L.cum = (int32_t)((uint32_t)(ws.efw[slot[i]] ? arc_vs(aid) : arc_ve(aid)) << LE_VID_SHIFT);   // start vertex
        }
      }
      nle += tot;
    }
  }
  g.sync();

  PHASE_MARK(6);
  // ---- 6. hole contours: cap arcs chained around the exposed sphere (lane 0) --------
  bool anycap = false;   // nodes without cap arcs (the sphere fully covered) have no holes
  if (status == 0 && d > 0) {
    #pragma unroll 1
    for (int i = lane; i < na; i += G) anycap = anycap || arc_lo(ws.arcs[i].ids) == 0;
    anycap = g.any(anycap);
  }
  if (status == 0 && d > 0 && anycap) {
    int st = 0;
    if (lane == 0) {
      uint64_t used = 0;   // MAXA <= 64 tracked per word below
      uint64_t usedw[(MAXA + 63) / 64];
      for (int i = 0; i < (MAXA + 63) / 64; i++) usedw[i] = 0;
      (void)used;
      for (int i = 0; i < na && !st; i++) {
        const ArcRec &Ai = ws.arcs[i];
        if (arc_lo(Ai.ids) != 0 || ((usedw[i >> 6] >> (i & 63)) & 1)) continue;
        if (nh >= MAXH) { st = LMM_NODE_ACAP; break; }
        ws.hoff[nh++] = nhe;
        int cur = i;
        int hb0 = arc_hi(Ai.ids);
        int hf0 = ws.sign[hb0] < 0;
        int start_v = hf0 ? arc_vs(Ai.ids) : arc_ve(Ai.ids);
        for (;;) {
          usedw[cur >> 6] |= 1ull << (cur & 63);
          const ArcRec &C = ws.arcs[cur];
          int hf = ws.sign[arc_hi(C.ids)] < 0;
          ws.he[nhe++] = (uint32_t)cur | ((uint32_t)hf << 16);
          int endv = hf ? arc_ve(C.ids) : arc_vs(C.ids);
          if (endv == start_v) break;
          int nxt = -1;
          for (int j = 0; j < na && nxt < 0; j++) {
            const ArcRec &Aj = ws.arcs[j];
            if (arc_lo(Aj.ids) != 0 || ((usedw[j >> 6] >> (j & 63)) & 1)) continue;
            int hj = ws.sign[arc_hi(Aj.ids)] < 0;
            if ((hj ? arc_vs(Aj.ids) : arc_ve(Aj.ids)) == endv) nxt = j;
          }
          if (nxt < 0) { st = LMM_NODE_HOLE; break; }
          cur = nxt;
        }
      }
      ws.hoff[nh] = nhe;
    }
    st = g.shfl(st, 0);
    nh = g.shfl(nh, 0);
    nhe = g.shfl(nhe, 0);
    if (st) status = st;
  }
  g.sync();

  PHASE_MARK(7);
  // ---- 7. write the node's slabs ----------------------------------------------------
  if (status == 0 && (nv > slab_cap(d, SLAB_V_K, SLAB_V_K0) || na > slab_cap(d, SLAB_A_K, SLAB_A_K0) ||
                      nle > slab_cap(d, SLAB_L_K, SLAB_L_K0) || nh > slab_cap(d, SLAB_H_K, SLAB_H_K0) ||
                      nhe > slab_cap(d, SLAB_HE_K, SLAB_HE_K0)))
    status = LMM_NODE_ACAP;
  if (status != 0) { nv = na = nle = nh = nhe = 0; }
  if (lane == 0)
    P.node_hdr[n] = make_int4(status | (d << 8), nv | (na << 16), nh | (nle << 16), nhe);
  const int64_t lb = slab_base(off, n, SLAB_L_K, SLAB_L_K0);
  const int64_t hb = slab_base(off, n, SLAB_H_K, SLAB_H_K0);
  const int64_t heb = slab_base(off, n, SLAB_HE_K, SLAB_HE_K0);
  #pragma unroll 1
  for (int q = lane; q < nle; q += G) P.loop[lb + q] = ws.le[q];
  #pragma unroll 1
  for (int k = lane; k < d; k += G)
    P.loop_hdr[off + k] = status == 0 ? make_int2(ws.lfirst[k + 1], ws.lcount[k + 1]) : make_int2(0, 0);
  #pragma unroll 1
  for (int h = lane; h < nh; h += G) P.hole_hdr[hb + h] = make_int2(ws.hoff[h], ws.hoff[h + 1] - ws.hoff[h]);
  #pragma unroll 1
  for (int q = lane; q < nhe; q += G) { HoleEnt he; he.arc_fwd = ws.he[q]; he.cum = 0; P.hole_ent[heb + q] = he; }
  PHASE_MARK(8);
  g.sync();
}

template <int PART, int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
struct PartWS;
template <int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
struct PartWS<0, G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH> { using T = WS_A<MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>; };
template <int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
struct PartWS<1, G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH> { using T = WS_B<MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>; };
template <int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
struct PartWS<2, G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH> { using T = WS_C<MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>; };

#ifndef LMM_MM_PREFETCH_PART
#define LMM_MM_PREFETCH_PART 2   // the part kernel with the next-node L2 prefetch (see metamesh_kernel)
#endif
#ifndef LMM_MM_MINB_A
#define LMM_MM_MINB_A 8
#endif
#ifndef LMM_MM_MINB_B
#define LMM_MM_MINB_B 5
#endif
#ifndef LMM_MM_MINB_C
#define LMM_MM_MINB_C 1
#endif
template <int PART, int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
__global__ void __launch_bounds__(128, PART == 0 ? LMM_MM_MINB_A : (PART == 1 ? LMM_MM_MINB_B : LMM_MM_MINB_C))
metamesh_kernel(MMParams P) {
  using WS = typename PartWS<PART, G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto block = cg::this_thread_block();
  cg::thread_block_tile<G> g = cg::tiled_partition<G>(block);
  const int gid_in_block = threadIdx.x / G;
  WS &ws = reinterpret_cast<WS *>(smem_raw)[gid_in_block];
  const int groups_per_block = blockDim.x / G;
  const int gid = blockIdx.x * groups_per_block + gid_in_block;
  const int ngroups = gridDim.x * groups_per_block;
  // part C reads the node's side records, vertices and arcs written by parts A/B long before:
  // the next node's lines are prefetched towards L2 one node ahead (its id and CSR offsets are
  // loaded two nodes ahead, so neither waits).  Measured: part C only (part B as well was
  // slower on octet100: 53.1 vs 55.0 ms meta-mesh; stoch290 300.8 ms either way).
  int nx = -1, offx = 0, dx = 0;   // node i + ngroups of the coming iteration i
  if (PART == LMM_MM_PREFETCH_PART && gid + ngroups < P.n_list) {
    nx = P.node_list[gid + ngroups];
    offx = P.csr_off[nx];
    dx = P.csr_off[nx + 1] - offx;
  }
  for (int i = gid; i < P.n_list; i += ngroups) {
    if constexpr (PART == LMM_MM_PREFETCH_PART) {
      if (nx >= 0) {
        const int ls = (80 * dx + 127) / 128 + 1, lv = (32 * dx + 32 + 127) / 128 + 1;
        const int la = PART == 2 ? (48 * (3 * dx + 2) + 127) / 128 + 1 : 0;
        const char *ps = reinterpret_cast<const char *>(P.side + 5 * (int64_t)offx);
        const char *pv = reinterpret_cast<const char *>(P.vert + slab_base(offx, nx, SLAB_V_K, SLAB_V_K0));
        const char *pa = reinterpret_cast<const char *>(P.arc + slab_base(offx, nx, SLAB_A_K, SLAB_A_K0));
        for (int k = g.thread_rank(); k < ls + lv + la + 1; k += G) {
          const char *q = k < ls ? ps + 128 * k : (k < ls + lv ? pv + 128 * (k - ls) : (k < ls + lv + la ? pa + 128 * (k - ls - lv)
                                                                                                         : reinterpret_cast<const char *>(P.state + nx)));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
        }
      }
      nx = -1;
      if (i + 2 * ngroups < P.n_list) {
        nx = P.node_list[i + 2 * ngroups];
        offx = P.csr_off[nx];
        dx = P.csr_off[nx + 1] - offx;
      }
    }
    if constexpr (PART == 0) part_a<G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>(g, ws, P, P.node_list[i]);
    else if constexpr (PART == 1) part_b<G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>(g, ws, P, P.node_list[i]);
    else part_c<G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>(g, ws, P, P.node_list[i]);
  }
}

// nodes of degree 0 (nothing to mesh), 32..63 (left for the spill kernel, spill.cu) and
// > 63 (outside the model: sides 0..63 in one 64-bit tie mask)
__global__ void trivial_nodes_kernel(const int *csr_off, int N, int4 *node_hdr, int2 *loop_hdr) {
  int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  int d = csr_off[n + 1] - csr_off[n];
  if (d == 0) node_hdr[n] = make_int4(0, 0, 0, 0);
  else if (d > LMM_MAXD) {
    node_hdr[n] = make_int4((d > LMM_MAXD_SPILL ? LMM_NODE_DEGREE : LMM_NODE_SPILL) | (d << 8), 0, 0, 0);
    for (int k = 0; k < d; k++) loop_hdr[csr_off[n] + k] = make_int2(0, 0);
  }
}

template <int PART, int G, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
int launch_part(lmm_ctx *c, const MMParams &P) {
  using WS = typename PartWS<PART, G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>::T;
  const int threads = 128;
  const int groups = threads / G;
  size_t smem = sizeof(WS) * groups;
  auto kern = metamesh_kernel<PART, G, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  if (occ < 1) occ = 1;
  int64_t need = (P.n_list + groups - 1) / groups;
  int64_t grid = (int64_t)c->n_sm * occ;
  if (grid > need) grid = need;
  (c->n_launch++), kern<<<(unsigned)grid, threads, smem, c->stream>>>(P);
  CUDA_TRY(cudaGetLastError());
  return LMM_OK;
}

// GA, GB, GC: lanes per node in parts A, B, C (32 = warp per node, 16 = two nodes per warp)
template <int GA, int GB, int GC, int MAXS, int MAXJ, int MAXV, int MAXA, int MAXLE, int MAXH>
int launch_bucket(lmm_ctx *c, MMParams P) {
  if (P.n_list <= 0) return LMM_OK;
  int rc;
  if ((rc = launch_part<0, GA, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>(c, P))) return rc;
  if ((rc = launch_part<1, GB, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>(c, P))) return rc;
  return launch_part<2, GC, MAXS, MAXJ, MAXV, MAXA, MAXLE, MAXH>(c, P);
}
// lanes per node of each bucket's parts (tuning: -DLMM_B<b>_G<A|B|C>=16|32): degree <= 8 nodes
// go two per warp (the paper's packing of combinable work into one warp), higher degrees one
#ifndef LMM_B0_GA
#define LMM_B0_GA 16
#endif
#ifndef LMM_B0_GB
#define LMM_B0_GB 16
#endif
#ifndef LMM_B0_GC
#define LMM_B0_GC 16
#endif
#ifndef LMM_B1_GA
#define LMM_B1_GA 32
#endif
#ifndef LMM_B1_GB
#define LMM_B1_GB 32
#endif
#ifndef LMM_B1_GC
#define LMM_B1_GC 32
#endif
#ifndef LMM_B00_GN
#define LMM_B00_GN 8
#endif
#define LMM_B00_G LMM_B00_GN, LMM_B00_GN, LMM_B00_GN
#define LMM_B0_G LMM_B0_GA, LMM_B0_GB, LMM_B0_GC
#define LMM_B1_G LMM_B1_GA, LMM_B1_GB, LMM_B1_GC
#define LMM_B2_G 32, 32, 32
#define LMM_B3_G 32, 32, 32

}  // namespace

#ifdef LMM_PHASE_TIMING
extern "C" LMM_API int lmm_debug_ws_bytes(int bucket, int part) {
  switch (bucket * 3 + part) {
    case 0: return (int)sizeof(WS_A<LMM_B0_ARGS>);
    case 1: return (int)sizeof(WS_B<LMM_B0_ARGS>);
    case 2: return (int)sizeof(WS_C<LMM_B0_ARGS>);
    case 3: return (int)sizeof(WS_A<LMM_B1_ARGS>);
    case 4: return (int)sizeof(WS_B<LMM_B1_ARGS>);
    case 5: return (int)sizeof(WS_C<LMM_B1_ARGS>);
    case 6: return (int)sizeof(WS_A<LMM_B2_ARGS>);
    case 7: return (int)sizeof(WS_B<LMM_B2_ARGS>);
    case 8: return (int)sizeof(WS_C<LMM_B2_ARGS>);
    case 9: return (int)sizeof(WS_A<LMM_B3_ARGS>);
    case 10: return (int)sizeof(WS_B<LMM_B3_ARGS>);
    default: return (int)sizeof(WS_C<LMM_B3_ARGS>);
  }
}
#endif

int metamesh_run(lmm_ctx *c) {
  MMParams P;
  P.node = (const float4 *)c->node.p;
  P.csr_off = (const int *)c->csr_off.p;
  P.csr_ent = (const int2 *)c->csr_ent.p;
  P.ends = (const int2 *)c->ends.p;
  P.node_hdr = (int4 *)c->node_hdr.p;
  P.vert = (float4 *)c->vert.p;
  P.arc = (ArcRec *)c->arc.p;
  P.loop_hdr = (int2 *)c->loop_hdr.p;
  P.loop = (LoopRec *)c->loop.p;
  P.hole_hdr = (int2 *)c->hole_hdr.p;
  P.hole_ent = (HoleEnt *)c->hole_ent.p;
  {
    int rc0;
    if ((rc0 = dev_alloc(c->mm_side, sizeof(float4) * 5 * (2 * c->S + 1)))) return rc0;
    if ((rc0 = dev_alloc(c->mm_state, sizeof(int4) * (c->N + 1)))) return rc0;
  }
  // lexicographic triple and pair tables for up to LMM_MAXD + 1 sides: triples of n sides at
  // C(n,4), then (at PAIR0) pairs of n sides at C(n,3)
  constexpr int NS = LMM_MAXD + 1;
  constexpr int PAIR0 = NS * (NS - 1) * (NS - 2) * (NS - 3) / 24 + NS * (NS - 1) * (NS - 2) / 6;
  if (!c->tri3.p) {
    std::vector<uint32_t> t3;
    for (int n = 3; n <= NS; n++)
      for (int a = 0; a < n; a++)
        for (int b = a + 1; b < n; b++)
          for (int cc = b + 1; cc < n; cc++) t3.push_back((uint32_t)a | ((uint32_t)b << 8) | ((uint32_t)cc << 16));
    t3.resize(PAIR0, 0u);
    for (int n = 2; n <= NS; n++)
      for (int a = 0; a < n; a++)
        for (int b = a + 1; b < n; b++) t3.push_back((uint32_t)a | ((uint32_t)b << 8));
    int rc0;
    if ((rc0 = dev_alloc(c->tri3, sizeof(uint32_t) * t3.size()))) return rc0;
    CUDA_TRY(cudaMemcpy(c->tri3.p, t3.data(), sizeof(uint32_t) * t3.size(), cudaMemcpyHostToDevice));
  }
  P.tri3 = (const uint32_t *)c->tri3.p;
  P.pair2 = (const uint32_t *)c->tri3.p + PAIR0;
  P.side = (float4 *)c->mm_side.p;
  P.state = (int4 *)c->mm_state.p;
  const int *bn = (const int *)c->bucket_nodes.p;
  int rc;
  {
    KTimer t(c, LMM_K_METAMESH);
    if (c->N > 0) {
      (c->n_launch++), trivial_nodes_kernel<<<(unsigned)((c->N + 255) / 256), 256, 0, c->stream>>>(
          (const int *)c->csr_off.p, (int)c->N, (int4 *)c->node_hdr.p, (int2 *)c->loop_hdr.p);
      CUDA_TRY(cudaGetLastError());
    }
    // bucket b occupies bucket_nodes[bucket_off[b] .. bucket_off[b+1])
    auto sel = [&](int b) {
      P.node_list = bn + c->bucket_off[b];
      P.n_list = (int)(c->bucket_off[b + 1] - c->bucket_off[b]);
    };
    sel(0);
    if ((rc = launch_bucket<LMM_B00_G, LMM_B00_ARGS>(c, P))) return rc;
    sel(1);
    if ((rc = launch_bucket<LMM_B0_G, LMM_B0_ARGS>(c, P))) return rc;
    sel(2);
    if ((rc = launch_bucket<LMM_B1_G, LMM_B1_ARGS>(c, P))) return rc;
    sel(3);
    if ((rc = launch_bucket<LMM_B1_G, LMM_B1b_ARGS>(c, P))) return rc;
    sel(4);
    if ((rc = launch_bucket<LMM_B2_G, LMM_B2_ARGS>(c, P))) return rc;
    sel(5);
    if ((rc = launch_bucket<LMM_B3_G, LMM_B3_ARGS>(c, P))) return rc;
  }
  return LMM_OK;
}
