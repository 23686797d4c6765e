/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's sequential
 * kernels (BigGraphVis / commviz).  Used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg as the CHECKER and the
 * CPU baseline.  Never linked into or called by the product package.
 *
 * Each function restates one numba kernel of the reference; the citation is
 * the reference file:line (C/ = /root/reference/pkg/src/commviz/).
 * Arithmetic is int64 / float64 exactly as in the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* C/community.py:98-120  _scoda_pass: one sequential streaming pass.   */
/* ------------------------------------------------------------------ */
void orc_scoda_pass(const int64_t *edges, const int64_t *order, int64_t m,
                    int64_t thr, int tie, int64_t *deg, int64_t *lab) {
    for (int64_t k = 0; k < m; ++k) {
        int64_t e = order ? order[k] : k;
        int64_t u = edges[2 * e], v = edges[2 * e + 1];
        /* both counters read before either write (self-loop bumps once) */
        int64_t du = deg[u], dv = deg[v];
        du += (du <= thr);
        dv += (dv <= thr);
        deg[u] = du;
        deg[v] = dv;
        if (du > thr || dv > thr) continue;
        if (du < dv || (du == dv && tie == 0))
            lab[u] = lab[v];
        else if (dv < du || (du == dv && tie == 1))
            lab[v] = lab[u];
    }
}

/* ------------------------------------------------------------------ */
/* C/community.py:123-161  _resolve_labels: representative of x is the  */
/* minimum id on the cycle reached by following x -> lab[x].            */
/* Restated as: walk, colouring nodes with the walk id; a revisit of the */
/* current walk closes a cycle, a visit of an older walk reuses its rep. */
/* ------------------------------------------------------------------ */
int orc_resolve_labels(const int64_t *lab, int64_t n, int64_t *out) {
    int64_t *walk = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t *path = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    if (!walk || !path || !pos) { free(walk); free(path); free(pos); return -1; }
    for (int64_t i = 0; i < n; ++i) walk[i] = -1;
    for (int64_t s = 0; s < n; ++s) {
        if (walk[s] != -1) continue;
        int64_t len = 0, x = s, rep;
        for (;;) {
            if (walk[x] != -1 && walk[x] != s) { rep = out[x]; break; }
            if (walk[x] == s) {                 /* cycle path[pos[x]..len) */
                rep = x;
                for (int64_t t = pos[x]; t < len; ++t)
                    if (path[t] < rep) rep = path[t];
                break;
            }
            walk[x] = s; pos[x] = len; path[len++] = x;
            int64_t nx = lab[x];
            if (nx < 0 || nx >= n) { free(walk); free(path); free(pos); return -2; }
            if (nx == x) { rep = x; break; }
            x = nx;
        }
        for (int64_t t = 0; t < len; ++t) out[path[t]] = rep;
    }
    free(walk); free(path); free(pos);
    return 0;
}

/* ------------------------------------------------------------------ */
/* C/layout.py:85-94  _separation (coincident-point jitter).            */
/* ------------------------------------------------------------------ */
#define COINCIDE_EPS 1e-4
#define TWO_PI 6.283185307179586
static inline double sep(double *dx, double *dy, int64_t a, int64_t b) {
    double d2 = (*dx) * (*dx) + (*dy) * (*dy);
    if (d2 >= COINCIDE_EPS * COINCIDE_EPS) return sqrt(d2);
    int64_t h = (a * (int64_t)2654435761LL + b * (int64_t)40503) % (int64_t)65536;
    if (h < 0) h += 65536; /* numpy % is non-negative */
    double ang = TWO_PI * ((double)h / 65536.0);
    *dx = COINCIDE_EPS * cos(ang);
    *dy = COINCIDE_EPS * sin(ang);
    return COINCIDE_EPS;
}

/* ------------------------------------------------------------------ */
/* C/layout.py:97-212  _build_tree: sequential insertion quadtree.      */
/* Cell numbering follows insertion order, which the jitter key n+c     */
/* depends on, so the insertion procedure is restated step by step.     */
/* Returns cells used, or -1 when cap is too small.                     */
/* ------------------------------------------------------------------ */
#define MAX_DEPTH 40
typedef struct {
    int64_t cap;
    int64_t *children; /* cap*4 */
    int8_t *kind;      /* 0 empty 1 single 2 internal 3 aggregate */
    double *cmass, *csumx, *csumy, *cx, *cy, *chalf;
    int64_t *ccount, *leaf_body, *body_cell;
} orc_tree;

static int64_t new_child(orc_tree *t, int64_t *used, int64_t cur, int q) {
    if (*used >= t->cap) return -1;
    int64_t c = (*used)++;
    t->children[4 * cur + q] = c;
    double h = 0.5 * t->chalf[cur];
    t->cx[c] = t->cx[cur] + ((q & 1) ? h : -h);
    t->cy[c] = t->cy[cur] + ((q & 2) ? h : -h);
    t->chalf[c] = h;
    return c;
}

int64_t orc_build_tree(const double *pos, const double *mass, int64_t n,
                       int64_t cap, int64_t *children, int8_t *kind,
                       double *cmass, double *csumx, double *csumy,
                       int64_t *ccount, double *cx, double *cy, double *chalf,
                       int64_t *leaf_body, int64_t *body_cell) {
    orc_tree t = {cap, children, kind, cmass, csumx, csumy, cx, cy, chalf,
                  ccount, leaf_body, body_cell};
    for (int64_t c = 0; c < cap; ++c) {
        for (int q = 0; q < 4; ++q) children[4 * c + q] = -1;
        kind[c] = 0; cmass[c] = csumx[c] = csumy[c] = 0.0; ccount[c] = 0;
        cx[c] = cy[c] = chalf[c] = 0.0; leaf_body[c] = -1;
    }
    for (int64_t i = 0; i < n; ++i) body_cell[i] = -1;
    double minx = pos[0], maxx = pos[0], miny = pos[1], maxy = pos[1];
    for (int64_t i = 1; i < n; ++i) {
        double x = pos[2 * i], y = pos[2 * i + 1];
        if (x < minx) minx = x;
        if (x > maxx) maxx = x;
        if (y < miny) miny = y;
        if (y > maxy) maxy = y;
    }
    double half = 0.5 * fmax(maxx - minx, maxy - miny);
    if (!(half > 0.0)) half = 1e-6;
    half *= 1.0000001;
    cx[0] = 0.5 * (minx + maxx);
    cy[0] = 0.5 * (miny + maxy);
    chalf[0] = half;
    int64_t used = 1;
    for (int64_t b = 0; b < n; ++b) {
        double xb = pos[2 * b], yb = pos[2 * b + 1], mb = mass[b];
        int64_t cur = 0;
        int depth = 0;
        for (;;) {
            cmass[cur] += mb; csumx[cur] += mb * xb; csumy[cur] += mb * yb;
            ccount[cur] += 1;
            int k = kind[cur];
            if (k == 0) { kind[cur] = 1; leaf_body[cur] = b; body_cell[b] = cur; break; }
            if (k == 3) { body_cell[b] = cur; break; }
            if (k == 1) {
                if (depth >= MAX_DEPTH) { kind[cur] = 3; body_cell[b] = cur; break; }
                int64_t e = leaf_body[cur];
                kind[cur] = 2; leaf_body[cur] = -1;
                int qe = (pos[2 * e] >= cx[cur]) + 2 * (pos[2 * e + 1] >= cy[cur]);
                int64_t c = new_child(&t, &used, cur, qe);
                if (c < 0) return -1;
                kind[c] = 1; leaf_body[c] = e; body_cell[e] = c;
                cmass[c] = mass[e]; csumx[c] = mass[e] * pos[2 * e];
                csumy[c] = mass[e] * pos[2 * e + 1]; ccount[c] = 1;
            }
            int q = (xb >= cx[cur]) + 2 * (yb >= cy[cur]);
            int64_t nx = children[4 * cur + q];
            if (nx == -1) {
                nx = new_child(&t, &used, cur, q);
                if (nx < 0) return -1;
            }
            cur = nx;
            depth += 1;
        }
    }
    return used;
}

/* ------------------------------------------------------------------ */
/* C/layout.py:215-270  _repulsion_bh: per-body explicit-stack walk.    */
/* ------------------------------------------------------------------ */
void orc_repulsion_bh(const double *pos, const double *mass, int64_t n,
                      double kr, double theta, const int64_t *children,
                      const int8_t *kind, const double *cmass,
                      const double *csumx, const double *csumy,
                      const int64_t *ccount, const double *chalf,
                      const int64_t *leaf_body, const int64_t *body_cell,
                      double *out) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        double xi = pos[2 * i], yi = pos[2 * i + 1], mi = mass[i];
        double fx = 0.0, fy = 0.0;
        int64_t stack[4 * MAX_DEPTH + 8];
        int sp = 0;
        stack[sp++] = 0;
        while (sp > 0) {
            int64_t c = stack[--sp];
            if (ccount[c] == 0) continue;
            int k = kind[c];
            if (k == 1) {
                int64_t j = leaf_body[c];
                if (j == i) continue;
                double dx = xi - pos[2 * j], dy = yi - pos[2 * j + 1];
                double d = sep(&dx, &dy, i, j);
                double f = kr * mi * mass[j] / (d * d);
                fx += f * dx; fy += f * dy;
                continue;
            }
            double mc = cmass[c], mx = csumx[c], my = csumy[c];
            if (k == 3 && body_cell[i] == c) {
                mc -= mi; mx -= mi * xi; my -= mi * yi;
                if (mc <= 0.0) continue;
            }
            double dx = xi - mx / mc, dy = yi - my / mc;
            double d2 = dx * dx + dy * dy;
            double side = 2.0 * chalf[c];
            if (k == 3 || side * side < theta * theta * d2) {
                double d = sep(&dx, &dy, i, n + c);
                double f = kr * mi * mc / (d * d);
                fx += f * dx; fy += f * dy;
            } else {
                for (int q = 0; q < 4; ++q) {
                    int64_t ch = children[4 * c + q];
                    if (ch != -1) stack[sp++] = ch;
                }
            }
        }
        out[2 * i] = fx;
        out[2 * i + 1] = fy;
    }
}

/* C/layout.py:273-290  _repulsion_exact (theta <= 0). */
void orc_repulsion_exact(const double *pos, const double *mass, int64_t n,
                         double kr, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double fx = 0.0, fy = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double dx = pos[2 * i] - pos[2 * j], dy = pos[2 * i + 1] - pos[2 * j + 1];
            double d = sep(&dx, &dy, i, j);
            double f = kr * mass[i] * mass[j] / (d * d);
            fx += f * dx; fy += f * dy;
        }
        out[2 * i] = fx;
        out[2 * i + 1] = fy;
    }
}

/* C/layout.py:293-304  _attraction: linear springs accumulated into out. */
void orc_attraction(const double *pos, const int64_t *edges, int64_t m,
                    const double *weight, double sign, double *out) {
    for (int64_t e = 0; e < m; ++e) {
        int64_t u = edges[2 * e], v = edges[2 * e + 1];
        double dx = pos[2 * v] - pos[2 * u], dy = pos[2 * v + 1] - pos[2 * u + 1];
        double w = weight[e] * sign;
        out[2 * u] += w * dx; out[2 * u + 1] += w * dy;
        out[2 * v] -= w * dx; out[2 * v + 1] -= w * dy;
    }
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
