/* Per-ray kd walk simulator (study tool, fp64, exact): how many tiles and
 * node tests a single ray's walk costs under different child orders and
 * seeds.  Built and driven by tools/walk_sim.py. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int d, pt;
  int64_t n_nodes, n_tiles;
  const double* node_box; /* n_nodes x 2d (lo, hi) */
  const int32_t* node_range;
  const double* rec; /* kd-ordered rows, stride rs */
  int rs;
  int64_t n_rows;
} Tree;

static int use_lb = 1;
void set_lb(int v) { use_lb = v; }
static int use_joint = 0;
void set_joint(int v) { use_joint = v; }

/* exact min |y - z|^2 over y in box with u.y >= thr (KKT: y = clamp(z + lam u)) */
static double joint_d2(int d, const double* lo, const double* hi, const double* z, const double* u,
                       double thr) {
  double y[16], g = 0;
  for (int k = 0; k < d; ++k) { y[k] = fmin(fmax(z[k], lo[k]), hi[k]); g += u[k] * y[k]; }
  double a = 0, b = 1;
  if (g < thr) {
    for (;;) {  /* bracket */
      double gg = 0;
      for (int k = 0; k < d; ++k) gg += u[k] * fmin(fmax(z[k] + b * u[k], lo[k]), hi[k]);
      if (gg >= thr || b > 1e6) break;
      a = b; b *= 2;
    }
    for (int it = 0; it < 80; ++it) {
      double m = 0.5 * (a + b), gg = 0;
      for (int k = 0; k < d; ++k) gg += u[k] * fmin(fmax(z[k] + m * u[k], lo[k]), hi[k]);
      if (gg >= thr) b = m; else a = m;
    }
    for (int k = 0; k < d; ++k) y[k] = fmin(fmax(z[k] + b * u[k], lo[k]), hi[k]);
  }
  double s = 0;
  for (int k = 0; k < d; ++k) s += (y[k] - z[k]) * (y[k] - z[k]);
  return s;
}

typedef struct {
  double x[16], u[16];
  double thr, r02, s;
  double tb;
  int ib;
} Ray;

static double box_lb(const Tree* T, const Ray* r, int64_t node, double* d2z, double* umax_out) {
  const int d = T->d;
  const double* lo = T->node_box + node * 2 * d;
  const double* hi = lo + d;
  double dx = 0, dz = 0, um = 0;
  for (int k = 0; k < d; ++k) {
    double z = r->x[k] + (isfinite(r->tb) ? r->tb : 0) * r->u[k];
    double e = fmax(fmax(lo[k] - r->x[k], r->x[k] - hi[k]), 0);
    dx += e * e;
    double f = fmax(fmax(lo[k] - z, z - hi[k]), 0);
    dz += f * f;
    um += r->u[k] * (r->u[k] > 0 ? hi[k] : lo[k]);
  }
  *d2z = dz;
  *umax_out = um;
  double den = um - r->s;
  if (den <= 0) return INFINITY;
  double a = dx - r->r02;
  return a > 0 ? a / (2 * den) : 0.0;
}

static int need(const Tree* T, const Ray* r, int64_t node, double* lb, double* d2z) {
  double um;
  *lb = box_lb(T, r, node, d2z, &um);
  if (!(um > r->thr)) return 0;
  if (!isfinite(r->tb)) return 1;
  double rho2 = 0;
  const double* g = NULL;
  (void)g;
  /* rho^2 = |x_g - z|^2 = r02 - 2 t u.(x_g - x) + t^2, u.(x_g - x) = s - u.x */
  double ux = 0;
  for (int k = 0; k < T->d; ++k) ux += r->u[k] * r->x[k];
  rho2 = r->r02 - 2 * r->tb * (r->s - ux) + r->tb * r->tb;
  if (!(*d2z < rho2)) return 0;
  if (use_lb && *lb >= r->tb) return 0;
  if (use_joint) {
    double z[16];
    for (int k = 0; k < T->d; ++k) z[k] = r->x[k] + r->tb * r->u[k];
    const double* lo = T->node_box + node * 2 * T->d;
    if (!(joint_d2(T->d, lo, lo + T->d, z, r->u, r->thr) < rho2)) return 0;
  }
  return 1;
}

static int sub_rows = 0;        /* 0: off; else rows per sub-box */
static int64_t sub_needed = 0;  /* sub-boxes needed over the batch */
static int64_t sub_needed_sph = 0;  /* same groups with bounding SPHERES (centroid, max distance):
                                       the test |z - c| < rho + r is bilinear in (z, rho) x (c, r),
                                       i.e. it could run on the tensor core */
void set_sub(int v) { sub_rows = v; sub_needed = 0; sub_needed_sph = 0; }
int64_t get_sub_needed(void) { return sub_needed; }
int64_t get_sub_needed_sph(void) { return sub_needed_sph; }

static void count_subs(const Tree* T, const Ray* r, int64_t tile) {
  const int d = T->d;
  double ux = 0;
  for (int k = 0; k < d; ++k) ux += r->u[k] * r->x[k];
  const double rho2 = isfinite(r->tb) ? r->r02 - 2 * r->tb * (r->s - ux) + r->tb * r->tb : INFINITY;
  for (int s0 = 0; s0 < T->pt; s0 += sub_rows) {
    double lo[16], hi[16];
    int any = 0;
    for (int k = 0; k < d; ++k) { lo[k] = INFINITY; hi[k] = -INFINITY; }
    for (int j = s0; j < s0 + sub_rows; ++j) {
      const double* y = T->rec + (tile * T->pt + j) * T->rs;
      if (isinf(y[d])) continue;
      any = 1;
      for (int k = 0; k < d; ++k) { lo[k] = fmin(lo[k], y[k]); hi[k] = fmax(hi[k], y[k]); }
    }
    if (!any) continue;
    double dz = 0, um = 0;
    for (int k = 0; k < d; ++k) {
      double z = r->x[k] + (isfinite(r->tb) ? r->tb : 0) * r->u[k];
      double f = fmax(fmax(lo[k] - z, z - hi[k]), 0);
      dz += f * f;
      um += r->u[k] * (r->u[k] > 0 ? hi[k] : lo[k]);
    }
    if (um > r->thr && dz < rho2) ++sub_needed;
    /* bounding sphere of the same rows */
    double c[16], rad2 = 0, cz = 0, uc = 0;
    int cnt = 0;
    for (int k = 0; k < d; ++k) c[k] = 0;
    for (int j = s0; j < s0 + sub_rows; ++j) {
      const double* y = T->rec + (tile * T->pt + j) * T->rs;
      if (isinf(y[d])) continue;
      ++cnt;
      for (int k = 0; k < d; ++k) c[k] += y[k];
    }
    for (int k = 0; k < d; ++k) c[k] /= cnt;
    for (int j = s0; j < s0 + sub_rows; ++j) {
      const double* y = T->rec + (tile * T->pt + j) * T->rs;
      if (isinf(y[d])) continue;
      double q = 0;
      for (int k = 0; k < d; ++k) q += (y[k] - c[k]) * (y[k] - c[k]);
      rad2 = fmax(rad2, q);
    }
    for (int k = 0; k < d; ++k) {
      double z = r->x[k] + (isfinite(r->tb) ? r->tb : 0) * r->u[k];
      cz += (z - c[k]) * (z - c[k]);
      uc += r->u[k] * c[k];
    }
    const double rad = sqrt(rad2);
    if (uc + rad > r->thr && (!isfinite(rho2) || sqrt(cz) < sqrt(rho2) + rad)) ++sub_needed_sph;
  }
}

static void screen_tile(const Tree* T, Ray* r, int64_t tile) {
  const int d = T->d;
  if (sub_rows) count_subs(T, r, tile);
  for (int j = 0; j < T->pt; ++j) {
    int64_t i = tile * T->pt + j;
    const double* y = T->rec + i * T->rs;
    if (isinf(y[d])) continue;
    double q = 0, aa = 0;
    for (int k = 0; k < d; ++k) {
      q += r->u[k] * y[k];
      double a = r->x[k] - y[k];
      aa += a * a;
    }
    if (!(q > r->thr)) continue;
    double t = (aa - r->r02) / (2 * (q - r->s));
    if (t < r->tb || (t == r->tb && i < r->ib)) {
      r->tb = t;
      r->ib = (int)i;
    }
  }
}

/* order: 0 start-tile child first, 1 nearest (d2 to sphere centre) first,
 * 2 smallest lower bound first (DFS), 3 best-first priority queue by LB */
typedef struct { double key; int64_t node; } PQ;

static void pq_push(PQ* h, int* n, double key, int64_t node) {
  int i = (*n)++;
  h[i].key = key;
  h[i].node = node;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (h[p].key <= h[i].key) break;
    PQ t = h[p]; h[p] = h[i]; h[i] = t;
    i = p;
  }
}
static PQ pq_pop(PQ* h, int* n) {
  PQ top = h[0];
  h[0] = h[--(*n)];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, rr = l + 1, m = i;
    if (l < *n && h[l].key < h[m].key) m = l;
    if (rr < *n && h[rr].key < h[m].key) m = rr;
    if (m == i) break;
    PQ t = h[m]; h[m] = h[i]; h[i] = t;
    i = m;
  }
  return top;
}

int walk(const Tree* T, Ray* r, int order, int64_t start_tile, int64_t* tiles, int64_t* tests) {
  int64_t stk[256];
  int sp = 0;
  double lb, d2;
  *tiles = 0;
  *tests = 0;
  if (order == 3) {
    PQ* h = (PQ*)malloc(sizeof(PQ) * (2 * T->n_nodes + 4));
    int n = 0;
    ++*tests;
    if (need(T, r, 0, &lb, &d2)) pq_push(h, &n, lb, 0);
    while (n > 0) {
      PQ e = pq_pop(h, &n);
      if (use_lb && isfinite(r->tb) && e.key >= r->tb) break;
      int64_t node = e.node;
      const int32_t* rg = T->node_range + 2 * node;
      if (rg[1] - rg[0] == 1) {
        ++*tests;
        if (!need(T, r, node, &lb, &d2)) continue;
        ++*tiles;
        screen_tile(T, r, rg[0]);
        continue;
      }
      for (int c = 1; c <= 2; ++c) {
        int64_t ch = 2 * node + c;
        ++*tests;
        if (need(T, r, ch, &lb, &d2)) pq_push(h, &n, lb, ch);
      }
    }
    free(h);
    return 0;
  }
  ++*tests;
  if (need(T, r, 0, &lb, &d2)) stk[sp++] = 0;
  while (sp > 0) {
    int64_t node = stk[--sp];
    const int32_t* rg = T->node_range + 2 * node;
    if (rg[1] - rg[0] == 1) {
      /* re-test against the current sphere */
      ++*tests;
      if (!need(T, r, node, &lb, &d2)) continue;
      ++*tiles;
      screen_tile(T, r, rg[0]);
      continue;
    }
    int64_t l = 2 * node + 1, rr = 2 * node + 2;
    double lbl, lbr, d2l, d2r;
    *tests += 2;
    int nl = need(T, r, l, &lbl, &d2l), nr = need(T, r, rr, &lbr, &d2r);
    int left_first;
    if (order == 0) left_first = start_tile < T->node_range[2 * l + 1];
    else if (order == 1) left_first = d2l <= d2r;
    else left_first = lbl <= lbr;
    if (left_first) {
      if (nr) stk[sp++] = rr;
      if (nl) stk[sp++] = l;
    } else {
      if (nl) stk[sp++] = l;
      if (nr) stk[sp++] = rr;
    }
    if (sp > 250) return -1;
  }
  return 0;
}

/* batch driver: rays as arrays; seeds: tb0/ib0 per ray (inf/-1: none);
 * seed_tiles: n x ns tile ids screened first (-1 ends) */
int walk_batch(int d, int pt, int64_t n_nodes, int64_t n_tiles, const double* node_box,
               const int32_t* node_range, const double* rec, int rs, int64_t n_rows, int64_t n,
               const double* x, const double* u, const double* thr, const double* r02,
               const double* s, const int64_t* start_tile, const int64_t* seed_tiles, int nseed,
               const double* tb0, int order, int64_t* out_tiles, int64_t* out_tests,
               int32_t* out_idx, double* out_t) {
  Tree T = {d, pt, n_nodes, n_tiles, node_box, node_range, rec, rs, n_rows};
  for (int64_t k = 0; k < n; ++k) {
    Ray r;
    memcpy(r.x, x + k * d, sizeof(double) * d);
    memcpy(r.u, u + k * d, sizeof(double) * d);
    r.thr = thr[k];
    r.r02 = r02[k];
    r.s = s[k];
    r.tb = tb0 ? tb0[k] : INFINITY;
    r.ib = -1;
    int64_t st = 0;
    for (int j = 0; j < nseed; ++j) {
      int64_t tl = seed_tiles[k * nseed + j];
      if (tl >= 0) { screen_tile(&T, &r, tl); ++st; }
    }
    int64_t tiles, tests;
    if (walk(&T, &r, order, start_tile[k], &tiles, &tests)) return -1;
    out_tiles[k] = tiles + st;
    out_tests[k] = tests;
    out_idx[k] = r.ib;
    out_t[k] = r.tb;
  }
  return 0;
}
