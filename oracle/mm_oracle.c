/*
 * oracle/mm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  The product path (paper_2405_15197_b200/) never links, imports or
 * executes it, and shares no code with it.
 *
 * A plain, slow CPU oracle of the data-parallel hot path of Zou & Gao,
 * "Warp-centric GPU meta-meshing and fast triangulation of billion-scale lattice
 * structures":
 *   - per-node meta-mesh: vertices, circular/elliptical arcs, strut faces and
 *     hole (nodal-sphere) faces   (Sec. 4.1, Sec. 4.3.1, Eq. 7-9),
 *   - resolution-parametric triangulation: arc subdivision (Eq. 11-12), strut
 *     bands, hole fans (Eq. 13), Algorithm 1.
 *
 * Precision.  Every TOPOLOGY decision (which junctions are vertices, which arcs
 * exist, loop order, subdivision counts N, band stitching) is taken in IEEE
 * binary32 -- the paper's precision (Sec. 4.2.1: "each parameter occupies
 * a 4-byte floating-point number in GPU") -- with the operation order written
 * below (compile with -ffp-contract=off: no implicit fused multiply-add, no reassociation;
 * the explicit FMA() calls are the specification's, DESIGN.md Sec. 4 and reading R11).
 * GEOMETRY (vertex positions, ellipse parameters, triangle coordinates) is then
 * recomputed in binary64 for the topology so decided.  DESIGN.md "Readings" lists
 * every place where the paper is silent or garbled and the reading taken here.
 *
 * Built twice from this one source:
 *   liborc.so    -- the oracle: decisions in binary32 (real = float, atan2p polynomial);
 *   liborc64.so  -- -DORC_REAL64: the SAME algorithm with every decision in binary64
 *                   (real = double, libm atan2), optionally with a seeded relative jitter
 *                   of the side parameters.  It pins the binary32 decision specification:
 *                   tests/test_oracle_pins.py requires identical topology on every node
 *                   whose binary64 topology is stable under the jitter.
 *
 * Storage.  No capacity of the GPU kernels appears here: junctions, vertex clusters,
 * arcs and conic vertices are held in growable heap arrays.  The one limit is the tie
 * mask of a vertex, one 64-bit word over the sides (sphere + up to 63 struts): a node of
 * degree > 63 is ORC_E_DEGREE (reading R13).
 *
 * Model.  At a node with centre o and sphere radius R, each
 * incident strut k is a cone (cylinder when radii agree) tangent to the nodal
 * sphere.  With y = x - o, u_k the unit direction to the far node, L_k the strut
 * length and sin(beta_k) = (R - r_far)/L_k, the cone is the set where the tangent
 * length sqrt(|y|^2 - R^2) equals the affine function
 *        h_k(y) = w_k . y - e_k,   w_k = u_k / cos(beta_k),  e_k = R tan(beta_k).
 * Two such cones therefore meet in the plane h_a = h_b -- the auxiliary plane
 * P_{a,b} of PAPER.md Sec. 4.3.1 ("the intersection curve of two struts is a planar
 * conic section").  The sphere is side 0 with h_0 = 0.  A point of the lattice
 * boundary near the node satisfies sqrt(|y|^2-R^2) = max_k h_k(y); side k's face
 * is where h_k attains the max; arcs are where two sides tie; vertices where three
 * tie (the "triple junctions").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define ORC_MAXD 63          /* struts per node: sides 0..63 in one 64-bit tie mask */

#ifdef ORC_REAL64
typedef double real;
#define FMA fma
#define SQRT sqrt
#define FABS fabs
#define FLOOR floor
#define ATAN2P(y, x) atan2((y), (x))
#else
typedef float real;
#define FMA fmaf
#define SQRT sqrtf
#define FABS fabsf
#define FLOOR floorf
#define ATAN2P(y, x) orc_atan2p((y), (x))
#endif
typedef uint64_t smask;      /* bit k = side k */
#define BIT(k) ((smask)1 << (k))

#define TOL_REL ((real)1e-4f)    /* delta   = TOL_REL * R : tie tolerance              */
#define CTOL_REL ((real)1e-3f)   /* delta_c = CTOL_REL * R : vertex clustering radius  */
#define PI_R ((real)3.14159265358979324f)
#define TWO_PI_R ((real)6.28318530717958648f)
#define HALF_PI_F 1.57079632679489662f
#define PI_F 3.14159265358979324f
#define TWO_PI_F 6.28318530717958648f

enum {
  ORC_OK = 0, ORC_E_DEGREE = 1, ORC_E_STRUT = 2, ORC_E_JCAP = 3, ORC_E_CCAP = 4,
  ORC_E_ACAP = 5, ORC_E_CONIC = 6, ORC_E_UNREF = 7, ORC_E_CHAIN = 8,
  ORC_E_ANGLE = 9, ORC_E_EMPTY = 10, ORC_E_HOLE = 11, ORC_E_SHORT = 12,
  ORC_E_QCAP = 13
};
/* ORC_E_JCAP / CCAP / ACAP / QCAP are never produced (no storage capacities); the codes
 * stay reserved so that the status numbering matches include/lmm.h. */

/* ------------------------------------------------------------------------- */
/* decision arithmetic (binary32, or binary64 in liborc64), operation order fixed */
/* ------------------------------------------------------------------------- */
typedef struct { real x, y, z; } f3;
typedef struct { double x, y, z; } d3;

static inline f3 F3(real x, real y, real z) { f3 r = {x, y, z}; return r; }
static inline f3 f_sub(f3 a, f3 b) { return F3(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline f3 f_add(f3 a, f3 b) { return F3(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline f3 f_scl(f3 a, real s) { return F3(a.x * s, a.y * s, a.z * s); }
static inline f3 f_div(f3 a, real s) { return F3(a.x / s, a.y / s, a.z / s); }
/* dot and cross products with explicit fused multiply-adds (C99 fmaf, one
 * rounding each): dot = fma(a.z, b.z, fma(a.y, b.y, a.x b.x)), cross.x = fma(a.y, b.z, -(a.z b.y)) */
static inline real f_dot(f3 a, f3 b) { return FMA(a.z, b.z, FMA(a.y, b.y, a.x * b.x)); }
static inline f3 f_cross(f3 a, f3 b) {
  return F3(FMA(a.y, b.z, -(a.z * b.y)), FMA(a.z, b.x, -(a.x * b.z)), FMA(a.x, b.y, -(a.y * b.x)));
}
static inline f3 f_nrm(f3 a) { return f_div(a, SQRT(f_dot(a, a))); }

static inline d3 D3(double x, double y, double z) { d3 r = {x, y, z}; return r; }
static inline d3 d_sub(d3 a, d3 b) { return D3(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline d3 d_add(d3 a, d3 b) { return D3(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline d3 d_scl(d3 a, double s) { return D3(a.x * s, a.y * s, a.z * s); }
static inline d3 d_div(d3 a, double s) { return D3(a.x / s, a.y / s, a.z / s); }
static inline double d_dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline d3 d_cross(d3 a, d3 b) {
  return D3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline d3 d_nrm(d3 a) { return d_div(a, sqrt(d_dot(a, a))); }
static inline d3 d_of(f3 a) { return D3(a.x, a.y, a.z); }

/* Four-quadrant arc tangent in binary32 using only + - * / (so that both the
 * oracle and the kernel evaluate it bit-identically).  Cephes-style reduction
 * to [-tan(pi/8), tan(pi/8)] and its degree-9 odd polynomial; |err| ~ 1e-7 rad
 * (pinned against libm atan2 in tests/test_oracle_pins.py).  The binary64 build
 * decides with libm atan2 instead. */
float orc_atan2p(float y, float x) {
  float ax = fabsf(x), ay = fabsf(y);
  float mx = ax > ay ? ax : ay;
  float mn = ax > ay ? ay : ax;
  if (mx == 0.0f) return 0.0f;
  float r = mn / mx;
  float y0 = 0.0f;
  if (r > 0.41421356237309503f) { y0 = 0.78539816339744831f; r = (r - 1.0f) / (r + 1.0f); }
  float z = r * r;
  float p = ((8.05374449538e-2f * z - 1.38776856032e-1f) * z + 1.99777106478e-1f) * z - 3.33329491539e-1f;
  float a = y0 + (p * z * r + r);
  if (ay > ax) a = HALF_PI_F - a;
  if (x < 0.0f) a = PI_F - a;
  if (y < 0.0f) a = -a;
  return a;
}

/* growable heap array: ensure room for n+1 elements of size sz */
static int grow(void **p, int *cap, int n, size_t sz) {
  if (n < *cap) return 1;
  int nc = *cap ? 2 * *cap : 64;
  while (nc <= n) nc *= 2;
  void *q = realloc(*p, sz * (size_t)nc);
  if (!q) return 0;
  *p = q;
  *cap = nc;
  return 1;
}

/* ------------------------------------------------------------------------- */
/* lattice + CSR                                                              */
/* ------------------------------------------------------------------------- */
typedef struct {
  int32_t lo, hi, vs, ve;     /* sides (lo<hi, 0 = sphere), start/end vertex      */
  real t0, dt;                /* decision parameter range on the conic (t0, t0+dt) */
  real tmid;                  /* tangent length at the interval midpoint           */
  f3 o, a, b;                 /* decision conic v(t) = a sin t + b cos t + o      */
  d3 o64, a64, b64;           /* binary64 conic                                  */
  double t064, dt64;          /* binary64 parameter range                        */
} arc_t;

typedef struct {
  smask mask;                 /* sides tied at this vertex (bit k = side k)       */
  int32_t kind;               /* 0: junction cluster, 1: seam of a closed arc     */
  int32_t ja, jb, jc, jr;     /* representative triple and root (kind 0)          */
  int32_t seam_arc;           /* arc owning the seam (kind 1)                     */
  f3 y;                       /* decision position, node-local                    */
  d3 y64;                     /* binary64 position, node-local                    */
} vert_t;

typedef struct { int32_t arc, fwd; real phs, dph; } loop_t;
typedef struct { int32_t arc, fwd; } hole_t;

typedef struct {
  int32_t status, d, nv, na, nh;
  vert_t *v;
  arc_t *a;
  int32_t *loop_off;          /* [d+1] into le                                    */
  loop_t *le;
  int32_t *hole_off;          /* [nh+1] into he                                   */
  hole_t *he;
  int32_t done;
} node_mm;

typedef struct orc_lat {
  int64_t n_nodes, n_struts;
  float *xyz, *rad;
  int64_t *ends;
  int64_t *csr_off;           /* [n_nodes+1] */
  int64_t *csr_strut;         /* [2S] incident struts, ascending per node */
  node_mm *mm;                /* [n_nodes] */
  /* triangulation */
  double ce; real th0;
  int64_t *band_n;            /* [S][3]: nA, nB, kB (rotation) */
  int64_t *strut_tri_off;     /* [S+1] */
  int64_t *hole_base;         /* [n_nodes+1] global hole index of node's first hole */
  int64_t *hole_M;            /* [n_holes] */
  int64_t *hole_tri_off;      /* [n_holes+1], added to strut_tri_off[S] */
  d3 *hole_bp;                /* [n_holes] projected centre, node-local */
  int64_t n_tri;
  int32_t tri_ready;
  /* binary64 build only: relative jitter of the side parameters (0 = none) */
  double jitter;
  uint64_t jitter_seed;
} orc_lat;

static void node_free(node_mm *m) {
  free(m->v); free(m->a); free(m->loop_off); free(m->le); free(m->hole_off); free(m->he);
  memset(m, 0, sizeof(*m));
}

orc_lat *orc_create(const float *xyz, const float *rad, int64_t n_nodes,
                    const int64_t *ends, int64_t n_struts) {
  orc_lat *L = (orc_lat *)calloc(1, sizeof(orc_lat));
  L->n_nodes = n_nodes; L->n_struts = n_struts;
  L->xyz = (float *)malloc(sizeof(float) * 3 * (size_t)n_nodes + 4);
  L->rad = (float *)malloc(sizeof(float) * (size_t)n_nodes + 4);
  L->ends = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)n_struts + 8);
  memcpy(L->xyz, xyz, sizeof(float) * 3 * (size_t)n_nodes);
  memcpy(L->rad, rad, sizeof(float) * (size_t)n_nodes);
  memcpy(L->ends, ends, sizeof(int64_t) * 2 * (size_t)n_struts);
  /* CSR: node -> incident struts in ascending strut id (SPEC.md neighbors_at:
   * "deterministic ascending order").  Plain counting sort. */
  L->csr_off = (int64_t *)calloc((size_t)n_nodes + 1, sizeof(int64_t));
  for (int64_t s = 0; s < n_struts; s++) { L->csr_off[ends[2 * s] + 1]++; L->csr_off[ends[2 * s + 1] + 1]++; }
  for (int64_t n = 0; n < n_nodes; n++) L->csr_off[n + 1] += L->csr_off[n];
  L->csr_strut = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)n_struts + 8);
  int64_t *fill = (int64_t *)calloc((size_t)n_nodes + 1, sizeof(int64_t));
  for (int64_t s = 0; s < n_struts; s++)
    for (int e = 0; e < 2; e++) {
      int64_t n = ends[2 * s + e];
      L->csr_strut[L->csr_off[n] + fill[n]++] = s;
    }
  free(fill);
  L->mm = (node_mm *)calloc((size_t)n_nodes + 1, sizeof(node_mm));
  return L;
}

void orc_destroy(orc_lat *L) {
  if (!L) return;
  for (int64_t n = 0; n < L->n_nodes; n++) node_free(&L->mm[n]);
  free(L->mm); free(L->xyz); free(L->rad); free(L->ends); free(L->csr_off); free(L->csr_strut);
  free(L->band_n); free(L->strut_tri_off); free(L->hole_base); free(L->hole_M);
  free(L->hole_tri_off); free(L->hole_bp);
  free(L);
}

/* binary64 build: seeded relative jitter of every side parameter (w, e, u, s), eps = 0 off */
void orc_set_jitter(orc_lat *L, double eps, uint64_t seed) { L->jitter = eps; L->jitter_seed = seed; }

#ifdef ORC_REAL64
static double jit(const orc_lat *L, int64_t n, int k, int comp) {
  /* splitmix64 of (seed, node, side, component) -> uniform in [-1, 1) */
  uint64_t z = L->jitter_seed * 0x9E3779B97F4A7C15ull + (uint64_t)n * 0xBF58476D1CE4E5B9ull +
               (uint64_t)(k * 16 + comp) * 0x94D049BB133111EBull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

#endif

static inline f3 node_pos(const orc_lat *L, int64_t n) {
  return F3(L->xyz[3 * n], L->xyz[3 * n + 1], L->xyz[3 * n + 2]);
}

/* ------------------------------------------------------------------------- */
/* sides of a node                                                            */
/* ------------------------------------------------------------------------- */
typedef struct {
  f3 w; real e;         /* h(y) = w.y - e                                   */
  f3 u; real s, c, L;   /* direction, sin/cos of cone half-angle, length     */
  f3 as, e1, e2;        /* strut canonical frame (axis i0->i1)              */
  int64_t strut; int sign;
} side32;

typedef struct { d3 w; double e; d3 u; double s, c, L; d3 as, e1, e2; } side64;

/* Canonical strut frame: axis as = (p[i1]-p[i0])/|.|, e1 = nrm(as x ref) with ref
 * the coordinate axis least aligned with as, e2 = as x e1.  Computed identically
 * at both ends so the two end loops share one angle coordinate. */
static void strut_frame32(const orc_lat *L, int64_t s, f3 *as, f3 *e1, f3 *e2) {
  f3 D = f_sub(node_pos(L, L->ends[2 * s + 1]), node_pos(L, L->ends[2 * s]));
  *as = f_nrm(D);
  real ax = FABS(as->x), ay = FABS(as->y), az = FABS(as->z);
  f3 ref = (ax <= ay && ax <= az) ? F3(1, 0, 0) : (ay <= az ? F3(0, 1, 0) : F3(0, 0, 1));
  *e1 = f_nrm(f_cross(*as, ref));
  *e2 = f_cross(*as, *e1);
}

static void strut_frame64(const orc_lat *L, int64_t s, d3 *as, d3 *e1, d3 *e2) {
  f3 as32, e132, e232;
  strut_frame32(L, s, &as32, &e132, &e232);   /* reference axis choice as decided */
  d3 D = d_sub(d_of(node_pos(L, L->ends[2 * s + 1])), d_of(node_pos(L, L->ends[2 * s])));
  *as = d_nrm(D);
  real ax = FABS(as32.x), ay = FABS(as32.y), az = FABS(as32.z);
  d3 ref = (ax <= ay && ax <= az) ? D3(1, 0, 0) : (ay <= az ? D3(0, 1, 0) : D3(0, 0, 1));
  *e1 = d_nrm(d_cross(*as, ref));
  *e2 = d_cross(*as, *e1);
}

/* Side k of node n (Sec. 4.3.1 strut notation; the cone half-angle is
 * read as alpha = -arcsin((R - r_far)/L), the SPEC.md erratum of the printed
 * arccos, which gives alpha = 0 for cylinders as the paper states). */
static int build_sides32(const orc_lat *L, int64_t n, side32 *S, int *d_out) {
  int64_t b = L->csr_off[n], d = L->csr_off[n + 1] - b;
  *d_out = (int)d;
  if (d > ORC_MAXD) return ORC_E_DEGREE;
  f3 o = node_pos(L, n);
  real R = L->rad[n];
  memset(&S[0], 0, sizeof(side32));
  for (int k = 1; k <= d; k++) {
    int64_t s = L->csr_strut[b + k - 1];
    int64_t far = L->ends[2 * s] == n ? L->ends[2 * s + 1] : L->ends[2 * s];
    side32 *q = &S[k];
    f3 D = f_sub(node_pos(L, far), o);
    real Ln = SQRT(f_dot(D, D));
    if (!(Ln > 0)) return ORC_E_STRUT;
    q->u = f_div(D, Ln);
    q->s = (R - (real)L->rad[far]) / Ln;
    if (!(FABS(q->s) < (real)0.9f)) return ORC_E_STRUT;
    q->c = SQRT(1 - q->s * q->s);
    q->w = f_div(q->u, q->c);
    q->e = (R * q->s) / q->c;
    q->L = Ln;
    q->strut = s;
    q->sign = (L->ends[2 * s] == n) ? 1 : -1;
    strut_frame32(L, s, &q->as, &q->e1, &q->e2);
#ifdef ORC_REAL64
    if (L->jitter != 0.0) {
      const double j = L->jitter;
      q->w.x *= 1 + j * jit(L, n, k, 0); q->w.y *= 1 + j * jit(L, n, k, 1); q->w.z *= 1 + j * jit(L, n, k, 2);
      q->e += j * R * jit(L, n, k, 3);
      q->u.x *= 1 + j * jit(L, n, k, 4); q->u.y *= 1 + j * jit(L, n, k, 5); q->u.z *= 1 + j * jit(L, n, k, 6);
      q->s += j * jit(L, n, k, 7);
    }
#endif
  }
  return ORC_OK;
}

static void build_sides64(const orc_lat *L, int64_t n, side64 *S) {
  int64_t b = L->csr_off[n], d = L->csr_off[n + 1] - b;
  d3 o = d_of(node_pos(L, n));
  double R = L->rad[n];
  memset(&S[0], 0, sizeof(side64));
  for (int k = 1; k <= d; k++) {
    int64_t s = L->csr_strut[b + k - 1];
    int64_t far = L->ends[2 * s] == n ? L->ends[2 * s + 1] : L->ends[2 * s];
    side64 *q = &S[k];
    d3 D = d_sub(d_of(node_pos(L, far)), o);
    double Ln = sqrt(d_dot(D, D));
    q->u = d_div(D, Ln);
    q->s = (R - (double)L->rad[far]) / Ln;
    q->c = sqrt(1.0 - q->s * q->s);
    q->w = d_div(q->u, q->c);
    q->e = R * q->s / q->c;
    q->L = Ln;
    strut_frame64(L, s, &q->as, &q->e1, &q->e2);
  }
}

/* side function h_k(y) = w_k . y - e_k, the dot product as in Sec. 4.1 */
static inline real h32(const side32 *S, int k, f3 y) { return k == 0 ? 0 : f_dot(S[k].w, y) - S[k].e; }

/* ------------------------------------------------------------------------- */
/* triple junctions: points where h_a = h_b = h_c = sqrt(|y|^2 - R^2)         */
/* ------------------------------------------------------------------------- */
/* The line {h_a = h_b = h_c} is y = y0 + lam*mh (two plane equations
 * n1.y = q1, n2.y = q2 with n1 = w_a - w_b, n2 = w_a - w_c); substituting into
 * |y|^2 - R^2 = tau^2, tau = h_a(y), gives A lam^2 + 2 B' lam + C = 0. */
static int junction32(const side32 *S, real R, int a, int b, int c, f3 *y, real *tau) {
  f3 Wa = S[a].w, Wb = S[b].w, Wc = S[c].w;
  real Ea = S[a].e, Eb = S[b].e, Ec = S[c].e;
  if (a == 0) { Wa = F3(0, 0, 0); Ea = 0; }
  f3 n1 = f_sub(Wa, Wb), n2 = f_sub(Wa, Wc);
  real q1 = Ea - Eb, q2 = Ea - Ec;
  f3 m = f_cross(n1, n2);
  real mm = f_dot(m, m);
  real nn1 = f_dot(n1, n1), nn2 = f_dot(n2, n2);
  if (!(mm > ((real)1e-8f * nn1) * nn2)) return 0;
  f3 c1 = f_cross(n2, m), c2 = f_cross(m, n1);
  real imm = 1 / mm;
  /* the fused multiply-adds of the junction solve */
  f3 y0 = F3(FMA(q2, c2.x, q1 * c1.x) * imm, FMA(q2, c2.y, q1 * c1.y) * imm, FMA(q2, c2.z, q1 * c1.z) * imm);
  real iml = 1 / SQRT(mm);
  f3 mh = f_scl(m, iml);
  real tau0 = f_dot(Wa, y0) - Ea;
  real tau1 = f_dot(Wa, mh);
  real A = FMA(-tau1, tau1, (real)1);
  if (!(A > (real)1e-6f)) return 0;
  real Bp = FMA(-tau0, tau1, f_dot(y0, mh));
  real C = FMA(-tau0, tau0, FMA(-R, R, f_dot(y0, y0)));
  real disc = FMA(Bp, Bp, -(A * C));
  if (disc < 0) return 0;
  real sq = SQRT(disc);
  real iA = 1 / A;
  real lam[2] = {(-Bp - sq) * iA, (-Bp + sq) * iA};
  for (int r = 0; r < 2; r++) {
    y[r] = F3(FMA(mh.x, lam[r], y0.x), FMA(mh.y, lam[r], y0.y), FMA(mh.z, lam[r], y0.z));
    tau[r] = FMA(lam[r], tau1, tau0);
  }
  return 2;
}

static void junction64(const side64 *S, double R, int a, int b, int c, int root, d3 *y) {
  d3 Wa = a == 0 ? D3(0, 0, 0) : S[a].w, Wb = S[b].w, Wc = S[c].w;
  double Ea = a == 0 ? 0.0 : S[a].e, Eb = S[b].e, Ec = S[c].e;
  d3 n1 = d_sub(Wa, Wb), n2 = d_sub(Wa, Wc);
  double q1 = Ea - Eb, q2 = Ea - Ec;
  d3 m = d_cross(n1, n2);
  double mm = d_dot(m, m);
  d3 c1 = d_cross(n2, m), c2 = d_cross(m, n1);
  d3 y0 = d_div(d_add(d_scl(c1, q1), d_scl(c2, q2)), mm);
  d3 mh = d_div(m, sqrt(mm));
  double tau0 = d_dot(Wa, y0) - Ea, tau1 = d_dot(Wa, mh);
  double A = 1.0 - tau1 * tau1;
  double Bp = d_dot(y0, mh) - tau0 * tau1;
  double C = (d_dot(y0, y0) - R * R) - tau0 * tau0;
  double disc = Bp * Bp - A * C;
  if (disc < 0.0) disc = 0.0;
  double sq = sqrt(disc);
  double lam = root == 0 ? (-Bp - sq) / A : (-Bp + sq) / A;
  *y = d_add(y0, d_scl(mh, lam));
}

/* ------------------------------------------------------------------------- */
/* conics: PAPER.md Eq. 7 (strut-plane ellipse) and the end-section circle    */
/* ------------------------------------------------------------------------- */
/* Strut a's ellipse in the auxiliary plane P_{a,b} (Eq. 7).  In node-local
 * coordinates v_i^0 = 0, d = -u_a (from v^1 towards v^0), r_i^0 = R,
 * Rot(d', alpha) d = cos(alpha) d + sin(alpha) (d' x d) with alpha = -beta.
 * Returns 0 when the section is not a bounded ellipse. */
static int ellipse32(const side32 *S, real R, int a, int b, f3 *o, f3 *av, f3 *bv) {
  const side32 *A = &S[a];
  f3 N = f_sub(A->w, S[b].w);
  real inl = 1 / SQRT(f_dot(N, N));
  f3 n = f_scl(N, inl);
  real pc = (A->e - S[b].e) * inl;
  f3 p = f_scl(n, pc);
  real s = A->s, c = A->c;
  if (!(FABS(f_dot(n, A->u)) > FABS(s) + (real)1e-3f)) return 0;
  f3 d = F3(-A->u.x, -A->u.y, -A->u.z);
  f3 dp = f_cross(d, n);
  real dpl2 = f_dot(dp, dp);
  f3 r_;
  if (dpl2 > (real)1e-12f) { dp = f_scl(dp, 1 / SQRT(dpl2)); r_ = f_cross(dp, d); }
  else r_ = A->e1;
  f3 g1 = F3(c * d.x - s * r_.x, c * d.y - s * r_.y, c * d.z - s * r_.z);
  f3 g2 = F3(c * d.x + s * r_.x, c * d.y + s * r_.y, c * d.z + s * r_.z);
  f3 F1 = F3(R * ((-s) * d.x - c * r_.x), R * ((-s) * d.y - c * r_.y), R * ((-s) * d.z - c * r_.z));
  f3 F2 = F3(R * ((-s) * d.x + c * r_.x), R * ((-s) * d.y + c * r_.y), R * ((-s) * d.z + c * r_.z));
  real k1 = f_dot(n, f_sub(p, F1)) / f_dot(n, g1);
  real k2 = f_dot(n, f_sub(p, F2)) / f_dot(n, g2);
  f3 E1 = f_add(F1, f_scl(g1, k1)), E2 = f_add(F2, f_scl(g2, k2));
  *o = f_scl(f_add(E1, E2), (real)0.5f);
  *av = f_scl(f_sub(E1, E2), (real)0.5f);
  real ad = f_dot(*av, d), aa = f_dot(*av, *av);
  real arg = 1 - (ad * ad) / ((c * c) * aa);
  if (arg < 0) arg = 0;
  real lam = SQRT(arg);
  *bv = f_scl(f_cross(*av, n), lam);
  if (!(f_dot(*bv, *bv) > (real)1e-12f * aa)) return 0;
  return 1;
}

static void ellipse64(const side64 *S, const side32 *S32, double R, int a, int b, d3 *o, d3 *av, d3 *bv) {
  const side64 *A = &S[a];
  d3 N = d_sub(A->w, S[b].w);
  double nl = sqrt(d_dot(N, N));
  d3 n = d_div(N, nl);
  d3 p = d_scl(n, (A->e - S[b].e) / nl);
  double s = A->s, c = A->c;
  d3 d = D3(-A->u.x, -A->u.y, -A->u.z);
  d3 dp = d_cross(d, n);
  double dpl2 = d_dot(dp, dp);
  d3 r_;
  /* degenerate-branch choice follows the decision arithmetic */
  f3 d32 = F3(-S32[a].u.x, -S32[a].u.y, -S32[a].u.z);
  f3 N32 = f_sub(S32[a].w, S32[b].w);
  f3 n32 = f_scl(N32, 1 / SQRT(f_dot(N32, N32)));
  f3 dp32 = f_cross(d32, n32);
  if (f_dot(dp32, dp32) > (real)1e-12f) { dp = d_div(dp, sqrt(dpl2)); r_ = d_cross(dp, d); }
  else r_ = A->e1;
  d3 g1 = d_sub(d_scl(d, c), d_scl(r_, s)), g2 = d_add(d_scl(d, c), d_scl(r_, s));
  d3 F1 = d_scl(d_sub(d_scl(d, -s), d_scl(r_, c)), R);
  d3 F2 = d_scl(d_add(d_scl(d, -s), d_scl(r_, c)), R);
  d3 E1 = d_add(F1, d_scl(g1, d_dot(n, d_sub(p, F1)) / d_dot(n, g1)));
  d3 E2 = d_add(F2, d_scl(g2, d_dot(n, d_sub(p, F2)) / d_dot(n, g2)));
  *o = d_scl(d_add(E1, E2), 0.5);
  *av = d_scl(d_sub(E1, E2), 0.5);
  double ad = d_dot(*av, d), aa = d_dot(*av, *av);
  double arg = 1.0 - (ad * ad) / (c * c * aa);
  if (arg < 0.0) arg = 0.0;
  *bv = d_scl(d_cross(*av, n), sqrt(arg));
}

/* End-section circle of strut b: the circle where its cone touches the nodal
 * sphere (Sec. 5 "the circle edge of the strut's end section"), read as
 * the tangency circle: centre R sin(beta) u, radius R cos(beta).  Parametrised by
 * the strut frame so that t is the angle around the strut axis. */
static void circle32(const side32 *S, real R, int b, f3 *o, f3 *av, f3 *bv) {
  real rs = R * S[b].s, rr = R * S[b].c;
  *o = f_scl(S[b].u, rs);
  *av = f_scl(S[b].e2, rr);
  *bv = f_scl(S[b].e1, rr);
}
static void circle64(const side64 *S, double R, int b, d3 *o, d3 *av, d3 *bv) {
  *o = d_scl(S[b].u, R * S[b].s);
  *av = d_scl(S[b].e2, R * S[b].c);
  *bv = d_scl(S[b].e1, R * S[b].c);
}

/* parameter t of point P on conic (o,a,b): sin t = Q.a/|a|^2, cos t = Q.b/|b|^2 */
static real conic_t32(f3 o, f3 av, f3 bv, f3 P, real *us, real *uc) {
  f3 Q = f_sub(P, o);
  real st = f_dot(Q, av) / f_dot(av, av);
  real ct = f_dot(Q, bv) / f_dot(bv, bv);
  real il = 1 / SQRT(st * st + ct * ct);
  *us = st * il; *uc = ct * il;
  return ATAN2P(st, ct);
}
static double conic_t64(d3 o, d3 av, d3 bv, d3 P) {
  d3 Q = d_sub(P, o);
  return atan2(d_dot(Q, av) / d_dot(av, av), d_dot(Q, bv) / d_dot(bv, bv));
}

/* ------------------------------------------------------------------------- */
/* validity tests                                                             */
/* ------------------------------------------------------------------------- */
/* junction of three struts: no other strut strictly above (tolerance delta),
 * and on the forward nappe (tau >= -delta, else the sphere is above). */
static int valid_strut_pt(const side32 *S, int d, smask excl, f3 y, real tau, real delta) {
  if (tau < -delta) return 0;
  for (int m = 1; m <= d; m++) {
    if (excl & BIT(m)) continue;
    if (h32(S, m, y) - tau > delta) return 0;
  }
  return 1;
}
/* sphere junction (sphere, b, c): no other strut above the sphere by more than delta
 * (tolerant, like strut junctions: near-coincident junctions then cluster into one
 * vertex of higher valence). */
static int valid_sphere_junction(const side32 *S, int d, smask excl, f3 y, real delta) {
  for (int m = 1; m <= d; m++) {
    if (excl & BIT(m)) continue;
    if (h32(S, m, y) > delta) return 0;
  }
  return 1;
}
/* a point of an end circle is exposed only if every other strut is below it by more
 * than delta: ties with the sphere go to the struts (zero-area holes vanish). */
static int valid_sphere_pt(const side32 *S, int d, smask excl, f3 y, real delta) {
  for (int m = 1; m <= d; m++) {
    if (excl & BIT(m)) continue;
    if (h32(S, m, y) > -delta) return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------------- */
/* per-node meta-mesh                                                         */
/* ------------------------------------------------------------------------- */
typedef struct { int a, b, c, r; f3 y; real tau; } junc_t;

/* scratch of one node (heap, grown on demand) */
typedef struct {
  junc_t *J; int capJ;
  int *lab, *cid; int capL;
  vert_t *V; int capV;
  arc_t *A; int capA;
  int *Q; real *tq, *us, *uc; int capQ;
} work_t;

static void work_free(work_t *w) {
  free(w->J); free(w->lab); free(w->cid); free(w->V); free(w->A);
  free(w->Q); free(w->tq); free(w->us); free(w->uc);
}

static int node_metamesh_at(orc_lat *L, int64_t n, int level) {
  node_mm *M = &L->mm[n];
  node_free(M);
  M->done = 1;
  side32 S[ORC_MAXD + 1];
  int d;
  int st = build_sides32(L, n, S, &d);
  M->d = d;
  M->loop_off = (int32_t *)calloc((size_t)d + 1, sizeof(int32_t));
  M->hole_off = (int32_t *)calloc(1, sizeof(int32_t));
  if (st != ORC_OK) { M->status = st; return st; }
  if (d == 0) return ORC_OK;
  real R = L->rad[n];
  real delta = TOL_REL * R, dc = (CTOL_REL * R) * (real)(1 << level);
  work_t W;
  memset(&W, 0, sizeof W);
#define FAIL(code) do { work_free(&W); M->status = (code); return M->status; } while (0)

  /* 1. junctions of every triple a<b<c of sides {0..d}, lexicographic order, root-minor */
  int nj = 0;
  for (int a = 0; a <= d; a++)
    for (int b = a + 1; b <= d; b++)
      for (int c = b + 1; c <= d; c++) {
        f3 y[2]; real tau[2];
        if (!junction32(S, R, a, b, c, y, tau)) continue;
        smask excl = BIT(a) | BIT(b) | BIT(c);
        for (int r = 0; r < 2; r++) {
          int ok = a == 0 ? valid_sphere_junction(S, d, excl, y[r], delta)
                          : valid_strut_pt(S, d, excl, y[r], tau[r], delta);
          if (!ok) continue;
          /* a vertex further along a strut than 0.45 of its length (x cos beta) lies where
           * the neighbouring node's meta-mesh takes over: the strut is too short for the model */
          int ks[3] = {a, b, c};
          for (int q = 0; q < 3; q++)
            if (ks[q] > 0 && tau[r] > (real)0.45f * (S[ks[q]].L * S[ks[q]].c)) FAIL(ORC_E_SHORT);
          if (!grow((void **)&W.J, &W.capJ, nj, sizeof(junc_t))) FAIL(ORC_E_JCAP);
          W.J[nj].a = a; W.J[nj].b = b; W.J[nj].c = c; W.J[nj].r = r; W.J[nj].y = y[r]; W.J[nj].tau = tau[r];
          nj++;
        }
      }

  /* 2. clustering: connected components of the graph "junctions within delta_c (max-norm)";
   *    a component is one vertex (of higher valence when several junctions coincide),
   *    positioned at and ordered by its lowest-index junction. */
  W.lab = (int *)malloc(sizeof(int) * (size_t)(nj + 1));
  W.cid = (int *)malloc(sizeof(int) * (size_t)(nj + 1));
  junc_t *J = W.J;
  int *lab = W.lab;
  for (int j = 0; j < nj; j++) lab[j] = j;
  for (int changed = 1; changed;) {
    changed = 0;
    for (int j = 0; j < nj; j++)
      for (int k = 0; k < nj; k++)
        if (lab[k] < lab[j] && FABS(J[j].y.x - J[k].y.x) <= dc && FABS(J[j].y.y - J[k].y.y) <= dc &&
            FABS(J[j].y.z - J[k].y.z) <= dc) { lab[j] = lab[k]; changed = 1; }
  }
  int nc = 0;
  for (int j = 0; j < nj; j++) {
    if (lab[j] == j) {
      if (!grow((void **)&W.V, &W.capV, nc, sizeof(vert_t))) FAIL(ORC_E_CCAP);
      W.cid[j] = nc;
      vert_t *V = &W.V[nc];
      V->kind = 0; V->ja = J[j].a; V->jb = J[j].b; V->jc = J[j].c; V->jr = J[j].r;
      V->y = J[j].y; V->mask = 0; V->seam_arc = -1;
      nc++;
    }
  }
  for (int j = 0; j < nj; j++) {
    smask bits = BIT(J[j].a) | BIT(J[j].b) | BIT(J[j].c);
    /* a strut junction at tangent length ~0 lies on the nodal sphere: it ties with side 0 */
    if (FABS(J[j].tau) <= delta) bits |= 1;
    W.V[W.cid[lab[j]]].mask |= bits;
  }
  int nv = nc;

  /* 3. arcs: for every pair of sides, walk the conic through its vertices.  A conic
   * carrying no vertex can only be one closed arc, which is then the whole loop of its
   * strut side(s): it is tested only when its strut sides appear in no vertex. */
  int na = 0;
  smask in_vertex = 0;
  for (int q = 0; q < nc; q++) in_vertex |= W.V[q].mask;
  for (int a = 0; a <= d; a++)
    for (int b = a + 1; b <= d; b++) {
      f3 o, av, bv;
      smask pm = BIT(a) | BIT(b);
      {
        int has = 0;
        for (int q = 0; q < nc && !has; q++) has = (W.V[q].mask & pm) == pm;
        smask strut_bits = a == 0 ? BIT(b) : pm;
        if (!has && (in_vertex & strut_bits)) continue;
      }
      if (a == 0) circle32(S, R, b, &o, &av, &bv);
      else if (!ellipse32(S, R, a, b, &o, &av, &bv)) {
        /* a pair whose plane section is unbounded cannot carry an arc only if no
         * vertex lies on it; otherwise the node is outside the model */
        for (int q = 0; q < nc; q++)
          if ((W.V[q].mask & pm) == pm) FAIL(ORC_E_CONIC);
        continue;
      }
      int nq = 0;
      for (int q = 0; q < nc; q++)
        if ((W.V[q].mask & pm) == pm) {
          if (nq >= W.capQ) {
            int cap = W.capQ;
            if (!grow((void **)&W.Q, &cap, nq, sizeof(int)) || !(W.tq = (real *)realloc(W.tq, sizeof(real) * (size_t)cap)) ||
                !(W.us = (real *)realloc(W.us, sizeof(real) * (size_t)cap)) || !(W.uc = (real *)realloc(W.uc, sizeof(real) * (size_t)cap)))
              FAIL(ORC_E_QCAP);
            W.capQ = cap;
          }
          W.Q[nq] = q;
          W.tq[nq] = conic_t32(o, av, bv, W.V[q].y, &W.us[nq], &W.uc[nq]);
          nq++;
        }
      int *Q = W.Q;
      real *tq = W.tq, *us = W.us, *uc = W.uc;
      /* insertion sort by (t, cluster index) */
      for (int i = 1; i < nq; i++)
        for (int j = i; j > 0 && (tq[j] < tq[j - 1] || (tq[j] == tq[j - 1] && Q[j] < Q[j - 1])); j--) {
          int ti = Q[j]; Q[j] = Q[j - 1]; Q[j - 1] = ti;
          real tf = tq[j]; tq[j] = tq[j - 1]; tq[j - 1] = tf;
          tf = us[j]; us[j] = us[j - 1]; us[j - 1] = tf;
          tf = uc[j]; uc[j] = uc[j - 1]; uc[j - 1] = tf;
        }
      int nint = nq == 0 ? 1 : nq;
      for (int i = 0; i < nint; i++) {
        real ms, mc, t0, dt;
        int vs, ve;
        if (nq == 0) { ms = 0; mc = 1; t0 = 0; dt = TWO_PI_R; vs = ve = -1; }
        else if (nq == 1) { ms = -us[0]; mc = -uc[0]; t0 = tq[0]; dt = TWO_PI_R; vs = ve = Q[0]; }
        else {
          int j = (i + 1) % nq;
          dt = j == 0 ? (tq[0] + TWO_PI_R) - tq[nq - 1] : tq[j] - tq[i];
          if (!(dt > 0)) FAIL(ORC_E_CHAIN);
          real sx = us[i] + us[j], sc = uc[i] + uc[j];
          real l2 = sx * sx + sc * sc;
          if (l2 > (real)1e-6f) {
            real l = SQRT(l2);
            ms = sx / l; mc = sc / l;
            if (dt > PI_R) { ms = -ms; mc = -mc; }
          } else { ms = uc[i]; mc = -us[i]; }
          t0 = tq[i]; vs = Q[i]; ve = Q[j];
        }
        f3 y = F3((o.x + av.x * ms) + bv.x * mc, (o.y + av.y * ms) + bv.y * mc, (o.z + av.z * ms) + bv.z * mc);
        real tmid = a == 0 ? 0 : h32(S, a, y);
        int ok = a == 0 ? valid_sphere_pt(S, d, pm, y, delta)
                        : valid_strut_pt(S, d, pm, y, tmid, delta);
        if (!ok) continue;
        if (!grow((void **)&W.A, &W.capA, na, sizeof(arc_t))) FAIL(ORC_E_ACAP);
        arc_t *E = &W.A[na];
        memset(E, 0, sizeof *E);
        E->lo = a; E->hi = b; E->t0 = t0; E->dt = dt; E->o = o; E->a = av; E->b = bv; E->tmid = tmid;
        if (vs < 0) {  /* closed conic without vertex: add its seam (t = 0) */
          if (!grow((void **)&W.V, &W.capV, nv, sizeof(vert_t))) FAIL(ORC_E_CCAP);
          vert_t *V = &W.V[nv];
          memset(V, 0, sizeof *V);
          V->kind = 1; V->mask = pm; V->seam_arc = na;
          V->y = F3(o.x + bv.x, o.y + bv.y, o.z + bv.z);
          vs = ve = nv++;
        }
        E->vs = vs; E->ve = ve;
        na++;
      }
    }
  vert_t *V = W.V;
  arc_t *A = W.A;

  /* An AMBIGUOUS strut-strut arc (a,b) -- tangent length at its midpoint within the tie
   * tolerance of the sphere -- whose two end vertices are also joined by the end-circle
   * arcs of a AND of b runs under a strictly exposed hole lune: the hole wins and the
   * arc is dropped (R10).  Seam references are renumbered. */
  {
    int w = 0;
    int *remap = (int *)malloc(sizeof(int) * (size_t)(na + 1));
    for (int i = 0; i < na; i++) {
      int drop = 0;
      if (A[i].lo > 0 && A[i].vs != A[i].ve && A[i].tmid < delta) {
        int ca = 0, cb = 0;
        for (int j = 0; j < na; j++) {
          if (A[j].lo != 0) continue;
          int same = (A[j].vs == A[i].vs && A[j].ve == A[i].ve) || (A[j].vs == A[i].ve && A[j].ve == A[i].vs);
          if (!same) continue;
          if (A[j].hi == A[i].lo) ca = 1;
          if (A[j].hi == A[i].hi) cb = 1;
        }
        drop = ca && cb;
      }
      remap[i] = drop ? -1 : w;
      if (!drop) A[w++] = A[i];
    }
    for (int q = nc; q < nv; q++) V[q].seam_arc = remap[V[q].seam_arc];
    free(remap);
    na = w;
  }

  if (getenv("ORC_DEBUG")) {
    for (int q = 0; q < nv; q++)
      fprintf(stderr, "node %lld v%d mask %llx y/R (%.5f %.5f %.5f)\n", (long long)n, q, (unsigned long long)V[q].mask,
              (double)(V[q].y.x / R), (double)(V[q].y.y / R), (double)(V[q].y.z / R));
    for (int i = 0; i < na; i++)
      fprintf(stderr, "node %lld arc%d (%d,%d) v%d->v%d t0=%.7f dt=%.7f\n", (long long)n, i, A[i].lo, A[i].hi, A[i].vs, A[i].ve,
              (double)A[i].t0, (double)A[i].dt);
  }
  /* every junction vertex must carry arcs */
  for (int q = 0; q < nc; q++) {
    int used = 0;
    for (int i = 0; i < na && !used; i++) used = A[i].vs == q || A[i].ve == q;
    if (!used) FAIL(ORC_E_UNREF);
  }

  /* 4. arc loops: one per strut end, ordered by angle around the strut axis
   *    (Sec. 4.1 "sequentially interconnected, forming an arc loop") */
  loop_t *LE = (loop_t *)malloc(sizeof(loop_t) * (size_t)(2 * na + 1));
  real *key = (real *)malloc(sizeof(real) * (size_t)(na + 1));
#undef FAIL
#define FAIL(code) do { free(LE); free(key); work_free(&W); M->status = (code); return M->status; } while (0)
  int nle = 0;
  for (int k = 1; k <= d; k++) {
    M->loop_off[k - 1] = nle;
    int beg = nle;
    f3 as = S[k].as, e1 = S[k].e1, e2 = S[k].e2;
    for (int i = 0; i < na; i++) {
      if (A[i].lo != k && A[i].hi != k) continue;
      int fwd = f_dot(f_cross(A[i].a, A[i].b), as) < 0;
      int vs = fwd ? A[i].vs : A[i].ve, ve = fwd ? A[i].ve : A[i].vs;
      real ps = ATAN2P(f_dot(V[vs].y, e2), f_dot(V[vs].y, e1));
      if (ps < 0) ps += TWO_PI_R;
      real dph;
      if (vs == ve) dph = TWO_PI_R;
      else {
        real pe = ATAN2P(f_dot(V[ve].y, e2), f_dot(V[ve].y, e1));
        if (pe < 0) pe += TWO_PI_R;
        dph = pe - ps;
        if (dph <= 0) dph += TWO_PI_R;
      }
      LE[nle].arc = i; LE[nle].fwd = fwd; LE[nle].phs = ps; LE[nle].dph = dph;
      key[nle - beg] = ps;
      nle++;
    }
    int cnt = nle - beg;
    if (cnt == 0) FAIL(ORC_E_EMPTY);
    for (int i = 1; i < cnt; i++)
      for (int j = i; j > 0 && (key[j] < key[j - 1] || (key[j] == key[j - 1] && LE[beg + j].arc < LE[beg + j - 1].arc)); j--) {
        loop_t t = LE[beg + j]; LE[beg + j] = LE[beg + j - 1]; LE[beg + j - 1] = t;
        real tf = key[j]; key[j] = key[j - 1]; key[j - 1] = tf;
      }
    if (getenv("ORC_DEBUG")) {
      fprintf(stderr, "node %lld strut side %d loop:", (long long)n, k);
      for (int i = 0; i < cnt; i++) {
        arc_t *E = &A[LE[beg + i].arc];
        fprintf(stderr, " [arc%d (%d,%d) v%d->v%d fwd%d ps=%.7f dph=%.7f]", LE[beg + i].arc, E->lo, E->hi, E->vs, E->ve,
                LE[beg + i].fwd, (double)LE[beg + i].phs, (double)LE[beg + i].dph);
      }
      fprintf(stderr, "\n");
    }
    real sum = 0;
    for (int i = 0; i < cnt; i++) {
      loop_t *x = &LE[beg + i], *y = &LE[beg + (i + 1) % cnt];
      int xe = x->fwd ? A[x->arc].ve : A[x->arc].vs;
      int ys = y->fwd ? A[y->arc].vs : A[y->arc].ve;
      if (xe != ys) FAIL(ORC_E_CHAIN);
      sum += x->dph;
    }
    if (FABS(sum - TWO_PI_R) > (real)1e-3f) FAIL(ORC_E_ANGLE);
    for (int i = 1; i < cnt; i++) LE[beg + i].phs = LE[beg + i - 1].phs + LE[beg + i - 1].dph;
  }
  M->loop_off[d] = nle;
  free(key);
  key = NULL;

  /* 5. holes: cap arcs chained around the exposed nodal sphere, traversed
   *    clockwise about each strut's outward direction (Sec. 5 holes) */
  hole_t *HE = (hole_t *)malloc(sizeof(hole_t) * (size_t)(na + 1));
  int32_t *hoff = (int32_t *)malloc(sizeof(int32_t) * (size_t)(na + 2));
  int nhe = 0, nh = 0;
  char *used = (char *)calloc((size_t)na + 1, 1);
  for (int i = 0; i < na; i++) {
    if (A[i].lo != 0 || used[i]) continue;
    hoff[nh++] = nhe;
    int cur = i;
    int hf0 = S[A[i].hi].sign < 0;
    int start_v = hf0 ? A[i].vs : A[i].ve;
    for (;;) {
      used[cur] = 1;
      int hf = S[A[cur].hi].sign < 0;
      HE[nhe].arc = cur; HE[nhe].fwd = hf; nhe++;
      int endv = hf ? A[cur].ve : A[cur].vs;
      if (endv == start_v) break;
      int nxt = -1;
      for (int j = 0; j < na && nxt < 0; j++) {
        if (A[j].lo != 0 || used[j]) continue;
        int hj = S[A[j].hi].sign < 0;
        if ((hj ? A[j].vs : A[j].ve) == endv) nxt = j;
      }
      if (nxt < 0) { free(HE); free(hoff); free(used); FAIL(ORC_E_HOLE); }
      cur = nxt;
    }
  }
  hoff[nh] = nhe;
  free(used);

  /* 6. binary64 geometry for the topology decided above */
  side64 S64[ORC_MAXD + 1];
  build_sides64(L, n, S64);
  double R64 = L->rad[n];
  for (int i = 0; i < na; i++) {
    arc_t *E = &A[i];
    if (E->lo == 0) circle64(S64, R64, E->hi, &E->o64, &E->a64, &E->b64);
    else ellipse64(S64, S, R64, E->lo, E->hi, &E->o64, &E->a64, &E->b64);
  }
  for (int q = 0; q < nv; q++) {
    if (V[q].kind == 0) junction64(S64, R64, V[q].ja, V[q].jb, V[q].jc, V[q].jr, &V[q].y64);
    else { arc_t *E = &A[V[q].seam_arc]; V[q].y64 = d_add(E->o64, E->b64); }
  }
  for (int i = 0; i < na; i++) {
    arc_t *E = &A[i];
    if (V[E->vs].kind == 1) { E->t064 = 0.0; E->dt64 = 2 * M_PI; continue; }
    double ts = conic_t64(E->o64, E->a64, E->b64, V[E->vs].y64);
    if (E->vs == E->ve) { E->t064 = ts; E->dt64 = 2 * M_PI; continue; }
    double te = conic_t64(E->o64, E->a64, E->b64, V[E->ve].y64);
    double dd = te - ts;
    /* pick the 2*pi branch closest to the decided span */
    double k = floor(((double)E->dt - dd) / (2 * M_PI) + 0.5);
    E->t064 = ts; E->dt64 = dd + 2 * M_PI * k;
  }

  M->nv = nv; M->na = na; M->nh = nh;
  M->v = V; M->a = A; M->le = LE; M->he = HE;
  W.V = NULL; W.A = NULL;
  work_free(&W);
  free(M->hole_off);
  M->hole_off = hoff;
  M->status = ORC_OK;
  return ORC_OK;
#undef FAIL
}

#ifndef ORC_MAX_LEVEL
#define ORC_MAX_LEVEL 4
#endif
static int node_metamesh(orc_lat *L, int64_t n) {
  int st = ORC_OK;
  for (int level = 0; level <= ORC_MAX_LEVEL; level++) {
    st = node_metamesh_at(L, n, level);
    if (!(st == ORC_E_CHAIN || st == ORC_E_HOLE || st == ORC_E_UNREF || st == ORC_E_ANGLE || st == ORC_E_EMPTY)) break;
    if (getenv("ORC_DEBUG")) fprintf(stderr, "node %lld: status %d at level %d\n", (long long)n, st, level);
  }
  return st;
}

/* compute the meta-mesh of selected nodes (nodes == NULL: all); a node in error keeps
 * only its status (no partial topology) */
int orc_metamesh(orc_lat *L, const int64_t *nodes, int64_t n_sel) {
  int64_t cnt = nodes ? n_sel : L->n_nodes;
  int64_t bad = 0;
  for (int64_t i = 0; i < cnt; i++) {
    int64_t n = nodes ? nodes[i] : i;
    if (node_metamesh(L, n) != ORC_OK) {
      node_mm *M = &L->mm[n];
      bad++;
      for (int k = 0; k <= M->d && M->loop_off; k++) M->loop_off[k] = 0;
      M->nv = M->na = M->nh = 0;
    }
  }
  L->tri_ready = 0;
  return (int)(bad > 2147483647 ? 2147483647 : bad);
}

/* Topology digest of a node: status, d, counts, tie masks, arc sides and endpoints, loop
 * order (arc, direction), hole contours -- no floating-point values.  FNV-1a 64. */
static uint64_t fnv(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; i++) { h ^= (v >> (8 * i)) & 0xff; h *= 0x100000001b3ull; }
  return h;
}
static uint64_t node_topo_hash(const node_mm *M) {
  uint64_t h = 0xcbf29ce484222325ull;
  h = fnv(h, (uint64_t)M->status); h = fnv(h, (uint64_t)M->d);
  if (M->status) return h;
  h = fnv(h, (uint64_t)M->nv); h = fnv(h, (uint64_t)M->na); h = fnv(h, (uint64_t)M->nh);
  for (int q = 0; q < M->nv; q++) h = fnv(h, M->v[q].mask);
  for (int i = 0; i < M->na; i++) {
    const arc_t *E = &M->a[i];
    h = fnv(h, (uint64_t)E->lo | ((uint64_t)E->hi << 16) | ((uint64_t)E->vs << 32) | ((uint64_t)E->ve << 48));
  }
  /* loops as cyclic sequences (their first entry, the smallest angle around the strut axis,
   * is a representation choice that flips where a vertex sits at angle 0): each rotated to
   * start at its lowest arc index */
  for (int k = 0; k <= M->d; k++) h = fnv(h, (uint64_t)M->loop_off[k]);
  for (int k = 0; k < M->d; k++) {
    const int b = M->loop_off[k], e = M->loop_off[k + 1], c = e - b;
    int r = 0;
    for (int i = 1; i < c; i++)
      if (M->le[b + i].arc < M->le[b + r].arc) r = i;
    for (int i = 0; i < c; i++) {
      const loop_t *x = &M->le[b + (r + i) % c];
      h = fnv(h, (uint64_t)x->arc | ((uint64_t)x->fwd << 32));
    }
  }
  for (int k = 0; k <= M->nh; k++) h = fnv(h, (uint64_t)(M->nh ? M->hole_off[k] : 0));
  int nhe = M->nh ? M->hole_off[M->nh] : 0;
  for (int i = 0; i < nhe; i++) h = fnv(h, (uint64_t)M->he[i].arc | ((uint64_t)M->he[i].fwd << 32));
  return h;
}

/* Meta-mesh of selected nodes, one at a time with nothing kept: status[i] and the
 * topology digest hash[i] (either may be NULL).  For scans of whole large lattices. */
void orc_metamesh_scan(orc_lat *L, const int64_t *nodes, int64_t n_sel, int32_t *status, uint64_t *hash) {
  for (int64_t i = 0; i < n_sel; i++) {
    int64_t n = nodes[i];
    node_metamesh(L, n);
    if (status) status[i] = L->mm[n].status;
    if (hash) hash[i] = node_topo_hash(&L->mm[n]);
    node_free(&L->mm[n]);
  }
  L->tri_ready = 0;
}

/* ------------------------------------------------------------------------- */
/* meta-mesh export                                                           */
/* ------------------------------------------------------------------------- */
int orc_node_counts(const orc_lat *L, int64_t n, int32_t *out /* status,d,nv,na,nh,nloop_entries,nhole_entries */) {
  const node_mm *M = &L->mm[n];
  out[0] = M->status; out[1] = M->d; out[2] = M->nv; out[3] = M->na; out[4] = M->nh;
  out[5] = M->loop_off ? M->loop_off[M->d] : 0;
  out[6] = (M->hole_off && M->nh) ? M->hole_off[M->nh] : 0;
  return M->done;
}

/* vertices: mask (64-bit), pos32[3] (decision arithmetic, as float), pos64[3] */
void orc_node_verts(const orc_lat *L, int64_t n, uint64_t *mask, float *pos32, double *pos64) {
  const node_mm *M = &L->mm[n];
  for (int q = 0; q < M->nv; q++) {
    mask[q] = M->v[q].mask;
    pos32[3 * q] = (float)M->v[q].y.x; pos32[3 * q + 1] = (float)M->v[q].y.y; pos32[3 * q + 2] = (float)M->v[q].y.z;
    pos64[3 * q] = M->v[q].y64.x; pos64[3 * q + 1] = M->v[q].y64.y; pos64[3 * q + 2] = M->v[q].y64.z;
  }
}

/* arcs: ints[4] = lo,hi,vs,ve ; f32[11] = t0,dt,o,a,b ; f64[11] = t0,dt,o,a,b */
void orc_node_arcs(const orc_lat *L, int64_t n, int32_t *ints, float *f32, double *f64) {
  const node_mm *M = &L->mm[n];
  for (int i = 0; i < M->na; i++) {
    const arc_t *E = &M->a[i];
    ints[4 * i] = E->lo; ints[4 * i + 1] = E->hi; ints[4 * i + 2] = E->vs; ints[4 * i + 3] = E->ve;
    float f[11] = {(float)E->t0, (float)E->dt, (float)E->o.x, (float)E->o.y, (float)E->o.z, (float)E->a.x, (float)E->a.y,
                   (float)E->a.z, (float)E->b.x, (float)E->b.y, (float)E->b.z};
    double g[11] = {E->t064, E->dt64, E->o64.x, E->o64.y, E->o64.z, E->a64.x, E->a64.y, E->a64.z, E->b64.x, E->b64.y, E->b64.z};
    memcpy(f32 + 11 * i, f, sizeof f);
    memcpy(f64 + 11 * i, g, sizeof g);
  }
}

/* loops: loop_off[d+1]; entries ints[2] = arc,fwd ; f32[2] = phs,dph */
void orc_node_loops(const orc_lat *L, int64_t n, int32_t *loop_off, int32_t *ints, float *f32) {
  const node_mm *M = &L->mm[n];
  for (int k = 0; k <= M->d; k++) loop_off[k] = M->loop_off ? M->loop_off[k] : 0;
  int ne = M->loop_off ? M->loop_off[M->d] : 0;
  for (int i = 0; i < ne; i++) {
    ints[2 * i] = M->le[i].arc; ints[2 * i + 1] = M->le[i].fwd;
    f32[2 * i] = (float)M->le[i].phs; f32[2 * i + 1] = (float)M->le[i].dph;
  }
}

/* holes: hole_off[nh+1]; entries ints[2] = arc,fwd */
void orc_node_holes(const orc_lat *L, int64_t n, int32_t *hole_off, int32_t *ints) {
  const node_mm *M = &L->mm[n];
  for (int h = 0; h <= M->nh; h++) hole_off[h] = M->nh ? M->hole_off[h] : 0;
  int ne = M->nh ? M->hole_off[M->nh] : 0;
  for (int i = 0; i < ne; i++) { ints[2 * i] = M->he[i].arc; ints[2 * i + 1] = M->he[i].fwd; }
}

void orc_csr(const orc_lat *L, int64_t *off, int64_t *strut) {
  memcpy(off, L->csr_off, sizeof(int64_t) * (size_t)(L->n_nodes + 1));
  memcpy(strut, L->csr_strut, sizeof(int64_t) * (size_t)(2 * L->n_struts));
}

/* ------------------------------------------------------------------------- */
/* triangulation (Sec. 5, Algorithm 1)                               */
/* ------------------------------------------------------------------------- */
/* Eq. 11: N = floor((t2 - t1) / (2 acos(1 - CE))) + 1, taken in binary32 with
 * th0 = (float)(2 acos(1 - CE)) evaluated once in binary64. */
static inline int arc_N(real dt, real th0) { return (int)FLOOR(dt / th0) + 1; }

float orc_theta0(double ce) { return (float)(2.0 * acos(1.0 - ce)); }
int orc_subdiv_count(float dt, float th0) { return arc_N(dt, th0); }
static real theta0_dec(double ce) { return (real)(2.0 * acos(1.0 - ce)); }

/* Eq. 12 point jj of arc (binary64): endpoints are the shared vertices exactly */
static d3 arc_point64(const node_mm *M, const arc_t *E, int N, int jj) {
  if (jj == 0) return M->v[E->vs].y64;
  if (jj == N) return M->v[E->ve].y64;
  double t = E->t064 + jj * (E->dt64 / N);
  return d_add(d_add(d_scl(E->a64, sin(t)), d_scl(E->b64, cos(t))), E->o64);
}

static int64_t loop_csr(const orc_lat *L, int64_t n, int64_t s) {
  for (int64_t i = L->csr_off[n]; i < L->csr_off[n + 1]; i++)
    if (L->csr_strut[i] == s) return i - L->csr_off[n];
  return -1;
}

typedef struct { int n; real *ang; d3 *pt; } ring_t;

/* the loop of strut s at node n as a ring of points (binary64) and stitch angles
 * (binary32: ang_j = phs + j * (dph / N) within each arc) */
static int loop_ring(const orc_lat *L, int64_t n, int64_t s, ring_t *rg, int want_pts) {
  const node_mm *M = &L->mm[n];
  rg->n = 0; rg->ang = NULL; rg->pt = NULL;
  if (M->status != ORC_OK || !M->done) return -1;
  int64_t k = loop_csr(L, n, s);
  int b = M->loop_off[k], e = M->loop_off[k + 1];
  int tot = 0;
  for (int i = b; i < e; i++) tot += arc_N(M->a[M->le[i].arc].dt, L->th0);
  rg->n = tot;
  rg->ang = (real *)malloc(sizeof(real) * (size_t)tot + 8);
  if (want_pts) rg->pt = (d3 *)malloc(sizeof(d3) * (size_t)tot);
  d3 on = d_of(node_pos(L, n));
  int p = 0;
  for (int i = b; i < e; i++) {
    const loop_t *x = &M->le[i];
    const arc_t *E = &M->a[x->arc];
    int N = arc_N(E->dt, L->th0);
    real step = x->dph / (real)N;
    for (int j = 0; j < N; j++) {
      rg->ang[p] = x->phs + (real)j * step;
      if (want_pts) rg->pt[p] = d_add(on, arc_point64(M, E, N, x->fwd ? j : N - j));
      p++;
    }
  }
  return 0;
}

static void ring_free(ring_t *r) { free(r->ang); free(r->pt); }

/* rotation of ring B so that it starts at its first point at/after A's start
 * angle (binary32 decisions) */
static int band_rotation(const ring_t *A, const ring_t *B, real *brel) {
  real a0 = A->ang[0];
  int k = 0;
  for (int j = 0; j < B->n; j++) {
    real r = B->ang[j] - a0;
    if (r < 0) r += TWO_PI_R;
    if (r >= TWO_PI_R) r -= TWO_PI_R;
    brel[j] = r;
    if (r < brel[k]) k = j;
  }
  return k;
}

static void tri_out(double *out, d3 p1, d3 p2, d3 p3) {
  d3 nn = d_cross(d_sub(p2, p1), d_sub(p3, p1));
  double l = sqrt(d_dot(nn, nn));
  if (l > 0) nn = d_div(nn, l);
  double v[12] = {nn.x, nn.y, nn.z, p1.x, p1.y, p1.z, p2.x, p2.y, p2.z, p3.x, p3.y, p3.z};
  memcpy(out, v, sizeof v);
}

/* band of strut s: merge rings A (end i0) and B (end i1) by stitch angle.
 * Writes triangles [from, to) of the band's nA+nB (out may be NULL). */
static void band_emit(const ring_t *A, const ring_t *B, int k, const real *brel, int64_t from, int64_t to, double *out) {
  int nA = A->n, nB = B->n;
  int i = 0, j = 0;
  for (int64_t t = 0; t < nA + nB && t < to; t++) {
    real an = (i + 1 < nA) ? A->ang[i + 1] - A->ang[0] : TWO_PI_R;
    real bn = (j + 1 < nB) ? brel[(j + 1 + k) % nB] : brel[k] + TWO_PI_R;
    int advA = i < nA && (j == nB || an <= bn);
    if (t >= from && out) {
      double *o = out + 12 * (t - from);
      if (advA) tri_out(o, A->pt[i % nA], A->pt[(i + 1) % nA], B->pt[(j + k) % nB]);
      else tri_out(o, A->pt[i % nA], B->pt[(j + 1 + k) % nB], B->pt[(j + k) % nB]);
    }
    if (advA) i++; else j++;
  }
}

/* hole ring (binary64), Eq. 13 fan centre */
static int hole_ring(const orc_lat *L, int64_t n, int h, d3 **pts, d3 *bp) {
  const node_mm *M = &L->mm[n];
  int b = M->hole_off[h], e = M->hole_off[h + 1];
  int tot = 0;
  for (int i = b; i < e; i++) tot += arc_N(M->a[M->he[i].arc].dt, L->th0);
  d3 *P = (d3 *)malloc(sizeof(d3) * (size_t)tot);
  int p = 0;
  for (int i = b; i < e; i++) {
    const arc_t *E = &M->a[M->he[i].arc];
    int N = arc_N(E->dt, L->th0);
    for (int j = 0; j < N; j++) P[p++] = arc_point64(M, E, N, M->he[i].fwd ? j : N - j);
  }
  /* Eq. 13: b = mean of contour vertices; b_project = (b-o)/|b-o| R + o.
   * Reading (R7): the direction is regularised by the contour's outward
   * (Newell) normal nu, b_project = R nrm(b + R nu/|nu|) + o, which equals Eq. 13's
   * direction for small holes and stays defined when b = o (free strut ends); a contour
   * without area (nu = 0) keeps Eq. 13's b - o. */
  d3 bsum = D3(0, 0, 0), nu = D3(0, 0, 0);
  for (int i = 0; i < tot; i++) {
    bsum = d_add(bsum, P[i]);
    nu = d_add(nu, d_cross(P[i], P[(i + 1) % tot]));
  }
  d3 bc = d_div(bsum, tot);
  double R = L->rad[n];
  /* a two-point contour (a lune of two one-segment arcs) has no area: nu = 0 exactly, and
   * Eq. 13's own direction b - o is used (reading R7) */
  const int flat = nu.x == 0.0 && nu.y == 0.0 && nu.z == 0.0;
  d3 dir = flat ? bc : d_add(bc, d_scl(d_nrm(nu), R));
  *bp = d_scl(d_nrm(dir), R);
  *pts = P;
  return tot;
}

/* Count pass: per-strut band sizes and rotations, per-hole sizes, offsets.
 * Global triangle order: struts ascending (band merge order), then nodes
 * ascending with their holes in order (fan i = 0..M-1). */
int64_t orc_triangulate(orc_lat *L, double ce) {
  L->ce = ce;
  L->th0 = theta0_dec(ce);
  free(L->band_n); free(L->strut_tri_off); free(L->hole_base); free(L->hole_M);
  free(L->hole_tri_off); free(L->hole_bp);
  int64_t S = L->n_struts;
  L->band_n = (int64_t *)calloc((size_t)S * 3, sizeof(int64_t));
  L->strut_tri_off = (int64_t *)calloc((size_t)S + 1, sizeof(int64_t));
  for (int64_t s = 0; s < S; s++) {
    ring_t A, B;
    int ra = loop_ring(L, L->ends[2 * s], s, &A, 0), rb = loop_ring(L, L->ends[2 * s + 1], s, &B, 0);
    if (ra == 0 && rb == 0 && A.n > 0 && B.n > 0) {
      real *brel = (real *)malloc(sizeof(real) * (size_t)B.n + 8);
      int k = band_rotation(&A, &B, brel);
      L->band_n[3 * s] = A.n; L->band_n[3 * s + 1] = B.n; L->band_n[3 * s + 2] = k;
      free(brel);
    }
    ring_free(&A); ring_free(&B);
    L->strut_tri_off[s + 1] = L->strut_tri_off[s] + L->band_n[3 * s] + L->band_n[3 * s + 1];
  }
  L->hole_base = (int64_t *)calloc((size_t)L->n_nodes + 1, sizeof(int64_t));
  for (int64_t n = 0; n < L->n_nodes; n++) {
    const node_mm *M = &L->mm[n];
    L->hole_base[n + 1] = L->hole_base[n] + ((M->done && M->status == ORC_OK) ? M->nh : 0);
  }
  int64_t H = L->hole_base[L->n_nodes];
  L->hole_M = (int64_t *)calloc((size_t)H + 1, sizeof(int64_t));
  L->hole_tri_off = (int64_t *)calloc((size_t)H + 1, sizeof(int64_t));
  L->hole_bp = (d3 *)calloc((size_t)H + 1, sizeof(d3));
  for (int64_t n = 0; n < L->n_nodes; n++) {
    const node_mm *M = &L->mm[n];
    if (!(M->done && M->status == ORC_OK)) continue;
    for (int h = 0; h < M->nh; h++) {
      d3 *P, bp;
      int tot = hole_ring(L, n, h, &P, &bp);
      free(P);
      int64_t g = L->hole_base[n] + h;
      /* a contour of two points (a lune of two one-segment arcs) has coincident chords: it
       * encloses no area at this chord error and gets no fan (reading R7) */
      L->hole_M[g] = tot == 2 ? 0 : tot;
      L->hole_bp[g] = bp;
    }
  }
  for (int64_t g = 0; g < H; g++) L->hole_tri_off[g + 1] = L->hole_tri_off[g] + L->hole_M[g];
  L->n_tri = L->strut_tri_off[S] + L->hole_tri_off[H];
  L->tri_ready = 1;
  return L->n_tri;
}

void orc_band_info(const orc_lat *L, int64_t *band_n /*[S][3]*/, int64_t *strut_off /*[S+1]*/) {
  memcpy(band_n, L->band_n, sizeof(int64_t) * 3 * (size_t)L->n_struts);
  memcpy(strut_off, L->strut_tri_off, sizeof(int64_t) * (size_t)(L->n_struts + 1));
}
int64_t orc_n_holes(const orc_lat *L) { return L->hole_base[L->n_nodes]; }
void orc_hole_info(const orc_lat *L, int64_t *hole_base /*[N+1]*/, int64_t *hole_M, double *bp /*[H][3]*/) {
  memcpy(hole_base, L->hole_base, sizeof(int64_t) * (size_t)(L->n_nodes + 1));
  int64_t H = L->hole_base[L->n_nodes];
  memcpy(hole_M, L->hole_M, sizeof(int64_t) * (size_t)H);
  for (int64_t g = 0; g < H; g++) { bp[3 * g] = L->hole_bp[g].x; bp[3 * g + 1] = L->hole_bp[g].y; bp[3 * g + 2] = L->hole_bp[g].z; }
}

/* triangles of strut s's band (binary64 absolute coordinates), all nA+nB of them */
int64_t orc_strut_triangles(const orc_lat *L, int64_t s, double *out) {
  ring_t A, B;
  int ra = loop_ring(L, L->ends[2 * s], s, &A, 1), rb = loop_ring(L, L->ends[2 * s + 1], s, &B, 1);
  int64_t cnt = 0;
  if (ra == 0 && rb == 0 && A.n > 0 && B.n > 0) {
    real *brel = (real *)malloc(sizeof(real) * (size_t)B.n + 8);
    int k = band_rotation(&A, &B, brel);
    band_emit(&A, &B, k, brel, 0, A.n + B.n, out);
    cnt = A.n + B.n;
    free(brel);
  }
  ring_free(&A); ring_free(&B);
  return cnt;
}

/* triangles of node n's holes (fans), in hole order */
int64_t orc_node_hole_triangles(const orc_lat *L, int64_t n, double *out) {
  const node_mm *M = &L->mm[n];
  if (!(M->done && M->status == ORC_OK)) return 0;
  d3 on = d_of(node_pos(L, n));
  int64_t cnt = 0;
  for (int h = 0; h < M->nh; h++) {
    d3 *P, bp;
    int tot = hole_ring(L, n, h, &P, &bp);
    if (tot == 2) { free(P); continue; }   /* flat lune: no fan (as orc_triangulate) */
    d3 apex = d_add(on, bp);
    for (int i = 0; i < tot; i++) {
      if (out) tri_out(out + 12 * cnt, apex, d_add(on, P[i]), d_add(on, P[(i + 1) % tot]));
      cnt++;
    }
    free(P);
  }
  return cnt;
}

/* all triangles in global order [first, first+count) */
int64_t orc_write_triangles(const orc_lat *L, int64_t first, int64_t count, double *out) {
  int64_t S = L->n_struts, w = 0, end = first + count;
  if (end > L->n_tri) end = L->n_tri;
  for (int64_t s = 0; s < S && w < end - first; s++) {
    int64_t b = L->strut_tri_off[s], e = L->strut_tri_off[s + 1];
    if (e <= first || b >= end) continue;
    int64_t m = e - b;
    double *tmp = (double *)malloc(sizeof(double) * 12 * (size_t)m);
    orc_strut_triangles(L, s, tmp);
    for (int64_t t = (b > first ? b : first); t < (e < end ? e : end); t++)
      memcpy(out + 12 * (t - first), tmp + 12 * (t - b), sizeof(double) * 12);
    free(tmp);
  }
  int64_t base = L->strut_tri_off[S];
  for (int64_t n = 0; n < L->n_nodes; n++) {
    int64_t g0 = L->hole_base[n], g1 = L->hole_base[n + 1];
    if (g0 == g1) continue;
    int64_t b = base + L->hole_tri_off[g0], e = base + L->hole_tri_off[g1];
    if (e <= first || b >= end) continue;
    double *tmp = (double *)malloc(sizeof(double) * 12 * (size_t)(e - b));
    orc_node_hole_triangles(L, n, tmp);
    for (int64_t t = (b > first ? b : first); t < (e < end ? e : end); t++)
      memcpy(out + 12 * (t - first), tmp + 12 * (t - b), sizeof(double) * 12);
    free(tmp);
  }
  return end - first;
}

/* ------------------------------------------------------------------------- */
/* building blocks exposed for the pins (binary64 unless noted)               */
/* ------------------------------------------------------------------------- */
/* Eq. 7 for a single cone: node at origin, radius R, strut direction u (unit),
 * sin(beta) = s; plane n.y = pc (n unit).  out = o[3], a[3], b[3]. */
void orc_eq7(const double *u, double s, double R, const double *n, double pc, const double *e1, double *out) {
  side64 S[2];
  memset(S, 0, sizeof S);
  S[1].u = D3(u[0], u[1], u[2]); S[1].s = s; S[1].c = sqrt(1 - s * s);
  S[1].w = d_div(S[1].u, S[1].c); S[1].e = R * s / S[1].c;
  S[1].e1 = D3(e1[0], e1[1], e1[2]);
  /* a fake second side whose auxiliary plane is the requested plane:
   * w_1 - w_2 = n * k, e_1 - e_2 = pc * k with k = 1 */
  S[0].w = d_sub(S[1].w, D3(n[0], n[1], n[2]));
  S[0].e = S[1].e - pc;
  side32 S32[2];
  memset(S32, 0, sizeof S32);
  S32[1].u = F3((float)u[0], (float)u[1], (float)u[2]);
  S32[1].w = F3((float)S[1].w.x, (float)S[1].w.y, (float)S[1].w.z);
  S32[0].w = F3((float)S[0].w.x, (float)S[0].w.y, (float)S[0].w.z);
  d3 o, a, b;
  side64 T[2] = {S[1], S[0]};
  side32 T32[2] = {S32[1], S32[0]};
  ellipse64(T, T32, R, 0, 1, &o, &a, &b);
  double v[9] = {o.x, o.y, o.z, a.x, a.y, a.z, b.x, b.y, b.z};
  memcpy(out, v, sizeof v);
}

/* auxiliary plane of two cones tangent to the sphere (centre 0, radius R):
 * n.y = pc with n = (w_a - w_b)/|w_a - w_b| (DESIGN.md Sec. 3 derivation). */
void orc_aux_plane(const double *ua, double sa, const double *ub, double sb, double R, double *n_out, double *pc) {
  double ca = sqrt(1 - sa * sa), cb = sqrt(1 - sb * sb);
  d3 wa = d_div(D3(ua[0], ua[1], ua[2]), ca), wb = d_div(D3(ub[0], ub[1], ub[2]), cb);
  d3 N = d_sub(wa, wb);
  double nl = sqrt(d_dot(N, N));
  d3 n = d_div(N, nl);
  n_out[0] = n.x; n_out[1] = n.y; n_out[2] = n.z;
  *pc = (R * sa / ca - R * sb / cb) / nl;
}

/* Eq. 8-9: the set {t : n.(v(t) - p) <= 0} on the conic v(t) = a sin t + b cos t + o,
 * as [lo, lo+len).  A = n.a, B = n.b, C = n.(p - o); A sin t + B cos t = rho cos(t - psi)
 * with rho = sqrt(A^2+B^2), psi = atan2(A, B) (the printed "t + tan^-1(B/A)" read as
 * this phase shift).  Returns 1 = FULL, 0 = EMPTY, 2 = range. */
int orc_eq9(const double *o, const double *a, const double *b, const double *n, const double *p, double *lo, double *len) {
  double A = n[0] * a[0] + n[1] * a[1] + n[2] * a[2];
  double B = n[0] * b[0] + n[1] * b[1] + n[2] * b[2];
  double C = n[0] * (p[0] - o[0]) + n[1] * (p[1] - o[1]) + n[2] * (p[2] - o[2]);
  double rho = sqrt(A * A + B * B);
  if (C >= rho) { *lo = 0; *len = 2 * M_PI; return 1; }
  if (C <= -rho) { *lo = 0; *len = 0; return 0; }
  double psi = atan2(A, B), ac = acos(C / rho);
  *lo = psi + ac;
  *len = 2 * M_PI - 2 * ac;
  return 2;
}
