/* Strut selection of the stochastic (Voronoi-style) lattice generator -- INPUT GENERATION
 * ONLY (no meta-meshing arithmetic).  Called from synth/lattices.py:stochastic().
 *
 * Nodes sit on a jittered side^3 grid (node id = (i*side + j)*side + k, position given by
 * the caller).  Nodes are visited in the caller's order (descending target degree, so the
 * high-degree hubs pick first); a node takes its nearest not-yet-joined neighbours from the
 * 5x5x5 surrounding grid cells, shortest first, while
 *   - both endpoints are below their target degree, and
 *   - the new strut is at least acos(cos_lim) away from every strut already at either end.
 * Deterministic for given inputs.  Build: gcc -O2 -shared -fPIC (synth/lattices.py). */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define MAXD 31
#define RAD 2
#define NC ((2 * RAD + 1) * (2 * RAD + 1) * (2 * RAD + 1))

typedef struct { double d2; int64_t b; } cand_t;

static void unit(const double *xyz, int64_t a, int64_t b, double u[3]) {
  double x = xyz[3 * b] - xyz[3 * a], y = xyz[3 * b + 1] - xyz[3 * a + 1], z = xyz[3 * b + 2] - xyz[3 * a + 2];
  double l = sqrt(x * x + y * y + z * z);
  u[0] = x / l; u[1] = y / l; u[2] = z / l;
}

/* 1 if direction u (from a) keeps the angle limit against every strut at a */
static int spread_ok(const double *xyz, const int32_t *nbr, const uint8_t *deg, int64_t a, const double u[3],
                     double cos_lim) {
  for (int m = 0; m < deg[a]; m++) {
    double w[3];
    unit(xyz, a, nbr[(int64_t)a * MAXD + m], w);
    if (u[0] * w[0] + u[1] * w[1] + u[2] * w[2] > cos_lim) return 0;
  }
  return 1;
}

int64_t stoch_struts(const double *xyz, int64_t side, const int32_t *target, const int64_t *order, double cos_lim,
                     int64_t max_struts, int64_t *ends) {
  int64_t N = side * side * side, S = 0;
  int32_t *nbr = (int32_t *)malloc(sizeof(int32_t) * (size_t)N * MAXD);
  uint8_t *deg = (uint8_t *)calloc((size_t)N, 1);
  if (!nbr || !deg) { free(nbr); free(deg); return -1; }
  cand_t c[NC];
  for (int64_t t = 0; t < N; t++) {
    int64_t a = order[t];
    if (deg[a] >= target[a]) continue;
    int64_t i = a / (side * side), j = (a / side) % side, k = a % side;
    int nc = 0;
    for (int64_t di = -RAD; di <= RAD; di++)
      for (int64_t dj = -RAD; dj <= RAD; dj++)
        for (int64_t dk = -RAD; dk <= RAD; dk++) {
          int64_t ii = i + di, jj = j + dj, kk = k + dk;
          if (ii < 0 || jj < 0 || kk < 0 || ii >= side || jj >= side || kk >= side) continue;
          int64_t b = (ii * side + jj) * side + kk;
          if (b == a || deg[b] >= target[b]) continue;
          int dup = 0;
          for (int m = 0; m < deg[a]; m++) dup |= nbr[a * MAXD + m] == b;
          if (dup) continue;
          double x = xyz[3 * b] - xyz[3 * a], y = xyz[3 * b + 1] - xyz[3 * a + 1], z = xyz[3 * b + 2] - xyz[3 * a + 2];
          cand_t e = {x * x + y * y + z * z, b};
          int p = nc++;   /* insertion sort: shortest first, ties by node id */
          while (p > 0 && (c[p - 1].d2 > e.d2 || (c[p - 1].d2 == e.d2 && c[p - 1].b > e.b))) { c[p] = c[p - 1]; p--; }
          c[p] = e;
        }
    for (int q = 0; q < nc && deg[a] < target[a]; q++) {
      int64_t b = c[q].b;
      if (deg[b] >= target[b]) continue;
      double u[3], v[3];
      unit(xyz, a, b, u);
      v[0] = -u[0]; v[1] = -u[1]; v[2] = -u[2];
      if (!spread_ok(xyz, nbr, deg, a, u, cos_lim) || !spread_ok(xyz, nbr, deg, b, v, cos_lim)) continue;
      if (S >= max_struts) { free(nbr); free(deg); return -2; }
      nbr[a * MAXD + deg[a]++] = (int32_t)b;
      nbr[b * MAXD + deg[b]++] = (int32_t)a;
      ends[2 * S] = a < b ? a : b;
      ends[2 * S + 1] = a < b ? b : a;
      S++;
    }
  }
  free(nbr);
  free(deg);
  return S;
}

/* Windowable variant (synth/lattices.py:stochastic_window): the same greedy on the zone of
 * layers [z0, z1) of an nx x ny x nz grid (node id (k*ny + j)*nx + i), degrees and neighbour
 * lists of the whole grid passed in and out so that a seam pass continues from the blocks'
 * state.  `order` lists the zone's nodes.  seam_k < 0: every pair of the zone may join;
 * seam_k >= 0: only pairs with one end below layer seam_k and one at or above it. */
int64_t stoch_zone(const double *xyz, int64_t nx, int64_t ny, int64_t nz, int64_t z0, int64_t z1, const int32_t *target,
                   const int64_t *order, double cos_lim, int64_t seam_k, uint8_t *deg, int32_t *nbr, int64_t max_struts,
                   int64_t *ends) {
  int64_t N = nx * ny * (z1 - z0), S = 0;
  cand_t c[NC];
  (void)nz;
  for (int64_t t = 0; t < N; t++) {
    int64_t a = order[t];
    if (deg[a] >= target[a]) continue;
    int64_t k = a / (nx * ny), j = (a / nx) % ny, i = a % nx;
    int nc = 0;
    for (int64_t dk = -RAD; dk <= RAD; dk++)
      for (int64_t dj = -RAD; dj <= RAD; dj++)
        for (int64_t di = -RAD; di <= RAD; di++) {
          int64_t ii = i + di, jj = j + dj, kk = k + dk;
          if (ii < 0 || jj < 0 || kk < z0 || ii >= nx || jj >= ny || kk >= z1) continue;
          if (seam_k >= 0 && ((k < seam_k) == (kk < seam_k))) continue;
          int64_t b = (kk * ny + jj) * nx + ii;
          if (b == a || deg[b] >= target[b]) continue;
          int dup = 0;
          for (int m = 0; m < deg[a]; m++) dup |= nbr[a * MAXD + m] == b;
          if (dup) continue;
          double x = xyz[3 * b] - xyz[3 * a], y = xyz[3 * b + 1] - xyz[3 * a + 1], z = xyz[3 * b + 2] - xyz[3 * a + 2];
          cand_t e = {x * x + y * y + z * z, b};
          int p = nc++;
          while (p > 0 && (c[p - 1].d2 > e.d2 || (c[p - 1].d2 == e.d2 && c[p - 1].b > e.b))) { c[p] = c[p - 1]; p--; }
          c[p] = e;
        }
    for (int q = 0; q < nc && deg[a] < target[a]; q++) {
      int64_t b = c[q].b;
      if (deg[b] >= target[b]) continue;
      double u[3], v[3];
      unit(xyz, a, b, u);
      v[0] = -u[0]; v[1] = -u[1]; v[2] = -u[2];
      if (!spread_ok(xyz, nbr, deg, a, u, cos_lim) || !spread_ok(xyz, nbr, deg, b, v, cos_lim)) continue;
      if (S >= max_struts) return -2;
      nbr[a * MAXD + deg[a]++] = (int32_t)b;
      nbr[b * MAXD + deg[b]++] = (int32_t)a;
      ends[2 * S] = a < b ? a : b;
      ends[2 * S + 1] = a < b ? b : a;
      S++;
    }
  }
  return S;
}
