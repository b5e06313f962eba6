/*
 * dem_oracle.c -- fp64 CPU oracle for the nonsmooth-DEM time step of
 * Pogulis & Servin, arXiv 2501.05300, TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
 * load this library.  It shares no code with the CUDA product path.
 *
 * Everything is plain fp64 in the paper's order: brute-force O(N^2) detection, the SPOOK
 * rows of the Hertz-mapped normal constraint, Coulomb disc and rolling ball projections,
 * a Jacobi projected-impulse sweep with mass splitting, symplectic position update.
 * Compiled with -ffp-contract=off so that the pair predicate has a fixed IEEE sequence.
 *
 * Parity pins: every function below is pinned by a test in tests/test_oracle_pins.py
 * (closed forms, SPEC worked examples, brute-force or library special cases); none is
 * "parity unpinned".  Readings R# are listed in DESIGN.md §3.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PI 3.14159265358979323846
#define WALL_KEY(w) (0xFFFFFFF0u + (uint32_t)(w))                 /* 2^32-16+w */
#define PLATE_KEY(p, b) (0xFFFFF000u + 16u * (uint32_t)(p) + (uint32_t)(b)) /* 2^32-4096+16p+b */

/* ---------------------------------------------------------------- small vector helpers */
static double dot3(const double *a, const double *b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
static void cross3(const double *a, const double *b, double *c)
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}
static double norm3(const double *a) { return sqrt(dot3(a, a)); }

/* ---------------------------------------------------------------- material */
void or_mass_inertia(double d, double rho, double *m, double *I)
{
    /* solid sphere: m = rho*pi*d^3/6, I = (2/5) m (d/2)^2 = m d^2/10 */
    double mm = rho * PI * d * d * d / 6.0;
    *m = mm;
    *I = mm * d * d / 10.0;
}

void or_contact_params(double da, double db, double Ea, double Eb, double nua, double nub,
                       double e_H, double *Estar, double *dstar, double *kn, double *eps_n)
{
    /* E* = [(1-nu_a^2)/E_a + (1-nu_b^2)/E_b]^-1, d* = (1/d_a + 1/d_b)^-1,
     * k_n = E* sqrt(d*)/3, eps_n = e_H/k_n.  A flat tool has infinite diameter. */
    double es = 1.0 / ((1.0 - nua * nua) / Ea + (1.0 - nub * nub) / Eb);
    double ds = (db > 0.0) ? 1.0 / (1.0 / da + 1.0 / db) : da;
    double k = es * sqrt(ds) / 3.0;
    *Estar = es;
    *dstar = ds;
    *kn = k;
    *eps_n = e_H / k;
}

/* ---------------------------------------------------------------- planner */
double or_profile_diameter(double d_min, double d_max, double gamma, double depth)
{
    /* Eq. 1: d(z) = d_min + gamma z for z < z_max = (d_max-d_min)/gamma, else d_max */
    if (gamma <= 0.0) return d_min;
    double z_max = (d_max - d_min) / gamma;
    return depth < z_max ? d_min + gamma * depth : d_max;
}

int32_t or_layer_schedule(double d_min, double d_max, double r, double eta,
                          double *d_out, double *z_out, int32_t cap)
{
    /* d_n = r d_{n-1}, thickness eta d_n, z_n = sum_{i<=n} eta d_i; the last layer is
     * clamped to d_max. */
    int32_t n = 0;
    double d = d_min, z = 0.0;
    if (r <= 1.0) {
        if (cap > 0) { d_out[0] = d_min; z_out[0] = eta * d_min; }
        return 1;
    }
    for (;;) {
        int last = d >= d_max * (1.0 - 1e-12);
        if (last) d = d_max;
        z += eta * d;
        if (n < cap) { d_out[n] = d; z_out[n] = z; }
        n++;
        if (last) break;
        d = r * d;
    }
    return n;
}

double or_contact_network_length(double d_min, double d_max, double r, double eta, double h)
{
    /* Eq. 10: n_d = eta ln(d_max/d_min)/ln r + (h - z_max)/d_max; uniform: h/d */
    if (d_max <= d_min || r <= 1.0) return h / d_max;
    double gamma = (r - 1.0) / (r * eta);
    double z_max = (d_max - d_min) / gamma;
    return eta * log(d_max / d_min) / log(r) + (h - z_max) / d_max;
}

int32_t or_solver_iterations(double n_d, double eps)
{
    /* Eq. 8: N_it = 0.1 n_d / eps, rounded up, at least 1 */
    double v = ceil(0.1 * n_d / eps - 1e-9);
    return v < 1.0 ? 1 : (int32_t)v;
}

double or_planned_timestep(double d, double eps, double rho, double sigma)
{
    /* Eq. 9: dt = 0.5 sqrt(eps d / a), a = 3 sigma / (2 rho d) */
    double a = 3.0 * sigma / (2.0 * rho * d);
    return 0.5 * sqrt(eps * d / a);
}

/* ---------------------------------------------------------------- detection */
typedef struct {
    uint64_t key;
    int64_t a;          /* particle index of body a */
    int64_t b;          /* particle index of body b, or -1 */
    int32_t kind;       /* 0 particle-particle, 1 wall, 2 plate */
    int32_t idx;        /* wall index or plate index */
    double n[3], delta;
} raw_contact;

typedef struct { raw_contact *v; int64_t n, cap; } raw_list;

static int push(raw_list *L, const raw_contact *c)
{
    if (L->n == L->cap) {
        int64_t nc = L->cap ? 2 * L->cap : 1024;
        raw_contact *nv = (raw_contact *)realloc(L->v, (size_t)nc * sizeof(raw_contact));
        if (!nv) return -1;
        L->v = nv;
        L->cap = nc;
    }
    L->v[L->n++] = *c;
    return 0;
}

static int cmp_raw(const void *x, const void *y)
{
    uint64_t a = ((const raw_contact *)x)->key, b = ((const raw_contact *)y)->key;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* Binning mode (SURVEY §8(c) "--binning": an independent CPU cell list, used for big-bed
 * timing).  Off by default; when on, the particle pairs are enumerated from a uniform grid of
 * cell 2 r_max instead of all N^2 pairs.  Every pair with d < r_a + r_b <= 2 r_max lies in
 * neighbouring cells, and each candidate goes through the same test as the brute force, so the
 * contact set, its values and (after the key sort) its order are identical; pinned against the
 * brute force by tests/test_oracle_pins.py. */
static int g_binning = 0;
void or_set_binning(int32_t on) { g_binning = on != 0; }

/* OpenMP threads of the sweeps (Jacobi is order-free).  Results do not depend on
 * the count: each contact is solved alone, each body sums its increments in contact order. */
#ifdef _OPENMP
#include <omp.h>
#endif
int32_t or_set_threads(int32_t n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* one particle pair (i, j): contact iff (dx^2+dy^2)+dz^2 < (r_a+r_b)^2 (reading R14) */
static int pair_test(const or_world *w, int64_t i, int64_t j, raw_list *L, int64_t *n_degen)
{
    int64_t a = i, b = j;
    if (w->gid[j] < w->gid[i]) { a = j; b = i; }
    double dx = w->x[3 * b + 0] - w->x[3 * a + 0];
    double dy = w->x[3 * b + 1] - w->x[3 * a + 1];
    double dz = w->x[3 * b + 2] - w->x[3 * a + 2];
    double d2 = (dx * dx + dy * dy) + dz * dz;
    double R = w->r[a] + w->r[b];
    if (!(d2 < R * R)) return 0;
    if (d2 == 0.0) { (*n_degen)++; return 0; }   /* coincident centres: flag+skip */
    double d = sqrt(d2);
    raw_contact c;
    c.key = ((uint64_t)w->gid[a] << 32) | (uint64_t)w->gid[b];
    c.a = a; c.b = b; c.kind = 0; c.idx = -1;
    c.n[0] = dx / d; c.n[1] = dy / d; c.n[2] = dz / d;
    c.delta = R - d;
    return push(L, &c);
}

/* particle pairs through the cell list; returns 1 if it cannot bin (non-finite input), so the
 * caller falls back to the brute force */
static int pairs_binned(const or_world *w, raw_list *L, int64_t *n_degen)
{
    const int64_t N = w->n;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY}, rmax = 0.0;
    for (int64_t i = 0; i < N; i++) {
        for (int k = 0; k < 3; k++) {
            const double x = w->x[3 * i + k];
            if (!isfinite(x)) return 1;
            if (x < lo[k]) lo[k] = x;
            if (x > hi[k]) hi[k] = x;
        }
        if (!isfinite(w->r[i])) return 1;
        if (w->r[i] > rmax) rmax = w->r[i];
    }
    double cell = 2.0 * rmax;
    int64_t n[3];
    for (;;) {                          /* at most ~8 cells per particle */
        int64_t tot = 1;
        for (int k = 0; k < 3; k++) { n[k] = (int64_t)floor((hi[k] - lo[k]) / cell) + 1; tot *= n[k]; }
        if (tot <= 8 * N + 64) break;
        cell *= 2.0;
    }
    const int64_t nc = n[0] * n[1] * n[2];
    int64_t *cnt = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
    int64_t *cid = (int64_t *)malloc((size_t)(N ? N : 1) * sizeof(int64_t));
    int64_t *lst = (int64_t *)malloc((size_t)(N ? N : 1) * sizeof(int64_t));
    if (!cnt || !cid || !lst) { free(cnt); free(cid); free(lst); return -1; }
    for (int64_t i = 0; i < N; i++) {
        int64_t c[3];
        for (int k = 0; k < 3; k++) {
            c[k] = (int64_t)floor((w->x[3 * i + k] - lo[k]) / cell);
            if (c[k] > n[k] - 1) c[k] = n[k] - 1;
        }
        cid[i] = c[0] + n[0] * (c[1] + n[1] * c[2]);
        cnt[cid[i] + 1]++;
    }
    for (int64_t c = 0; c < nc; c++) cnt[c + 1] += cnt[c];          /* cell starts */
    int64_t *fill = (int64_t *)malloc((size_t)nc * sizeof(int64_t));
    if (!fill) { free(cnt); free(cid); free(lst); return -1; }
    memcpy(fill, cnt, (size_t)nc * sizeof(int64_t));
    for (int64_t i = 0; i < N; i++) lst[fill[cid[i]]++] = i;
    free(fill);
    int rc = 0;
    for (int64_t i = 0; i < N && !rc; i++) {
        const int64_t cx = cid[i] % n[0], cy = (cid[i] / n[0]) % n[1], cz = cid[i] / (n[0] * n[1]);
        for (int64_t z = cz - 1; z <= cz + 1; z++)
            for (int64_t y = cy - 1; y <= cy + 1; y++)
                for (int64_t x = cx - 1; x <= cx + 1; x++) {
                    if (x < 0 || y < 0 || z < 0 || x >= n[0] || y >= n[1] || z >= n[2]) continue;
                    const int64_t c = x + n[0] * (y + n[1] * z);
                    for (int64_t t = cnt[c]; t < cnt[c + 1] && !rc; t++)
                        if (lst[t] > i) rc = pair_test(w, i, lst[t], L, n_degen);
                }
    }
    free(cnt); free(cid); free(lst);
    return rc;
}

/* All contacts of the current configuration, brute force (or binned), sorted by key. */
static int detect_all(const or_world *w, raw_list *L, int64_t *n_degen)
{
    const int64_t N = w->n;
    *n_degen = 0;
    int binned = 1;
    if (g_binning) {
        const int rc = pairs_binned(w, L, n_degen);
        if (rc < 0) return -1;
        if (rc == 1) { binned = 0; L->n = 0; *n_degen = 0; }
    } else {
        binned = 0;
    }
    if (!binned)
        for (int64_t i = 0; i < N; i++)
            for (int64_t j = i + 1; j < N; j++)
                if (pair_test(w, i, j, L, n_degen)) return -1;
    /* walls: s = (X-p).n_w < r -> n = -n_w, delta = r - s */
    for (int64_t i = 0; i < N; i++) {
        for (int32_t k = 0; k < w->n_walls; k++) {
            const or_wall *W = &w->walls[k];
            double s = ((w->x[3 * i] - W->p[0]) * W->n[0] + (w->x[3 * i + 1] - W->p[1]) * W->n[1])
                       + (w->x[3 * i + 2] - W->p[2]) * W->n[2];
            if (!(s < w->r[i])) continue;
            raw_contact c;
            c.key = ((uint64_t)w->gid[i] << 32) | (uint64_t)WALL_KEY(W->id);
            c.a = i; c.b = -1; c.kind = 1; c.idx = k;
            c.n[0] = -W->n[0]; c.n[1] = -W->n[1]; c.n[2] = -W->n[2];
            c.delta = w->r[i] - s;
            if (push(L, &c)) return -1;
        }
    }
    /* plate boxes: closest point q = clamp(X, lo, hi); contact iff |q-X|^2 < r^2 */
    for (int64_t i = 0; i < N; i++) {
        const double *X = &w->x[3 * i];
        for (int32_t p = 0; p < w->n_plates; p++) {
            const or_plate *P = &w->plates[p];
            for (int32_t bx = 0; bx < P->nbox; bx++) {
                double lo[3], hi[3], q[3], dq[3];
                for (int k = 0; k < 3; k++) {
                    lo[k] = P->pos[k] + P->lo[bx][k];
                    hi[k] = P->pos[k] + P->hi[bx][k];
                    q[k] = X[k] < lo[k] ? lo[k] : (X[k] > hi[k] ? hi[k] : X[k]);
                    dq[k] = q[k] - X[k];
                }
                double d2 = (dq[0] * dq[0] + dq[1] * dq[1]) + dq[2] * dq[2];
                double r = w->r[i];
                raw_contact c;
                c.key = ((uint64_t)w->gid[i] << 32) | (uint64_t)PLATE_KEY(p, bx);
                c.a = i; c.b = -1; c.kind = 2; c.idx = p;
                if (d2 > 0.0) {
                    if (!(d2 < r * r)) continue;
                    double d = sqrt(d2);
                    c.n[0] = dq[0] / d; c.n[1] = dq[1] / d; c.n[2] = dq[2] / d;
                    c.delta = r - d;
                } else {
                    /* centre inside the box (reading R19): exit through the nearest face;
                     * n points from the particle into the box, delta = r + depth */
                    double best = INFINITY; int bk = 0; double sg = 1.0;
                    for (int k = 0; k < 3; k++) {
                        double dl = X[k] - lo[k], dh = hi[k] - X[k];
                        if (dl < best) { best = dl; bk = k; sg = 1.0; }   /* exit via lo face: n = +e_k */
                        if (dh < best) { best = dh; bk = k; sg = -1.0; }  /* exit via hi face: n = -e_k */
                    }
                    c.n[0] = c.n[1] = c.n[2] = 0.0;
                    c.n[bk] = sg;
                    c.delta = r + best;
                }
                if (push(L, &c)) return -1;
            }
        }
    }
    qsort(L->v, (size_t)L->n, sizeof(raw_contact), cmp_raw);
    return 0;
}

int32_t or_detect(const or_world *w, const or_params *p, or_contact *out, int64_t cap,
                  int64_t *n_out, int64_t *n_degenerate)
{
    (void)p;
    raw_list L = {0, 0, 0};
    if (detect_all(w, &L, n_degenerate)) { free(L.v); return -1; }
    *n_out = L.n;
    if (L.n > cap) { free(L.v); return -1; }
    for (int64_t c = 0; c < L.n; c++) {
        out[c].key = L.v[c].key;
        memcpy(out[c].n, L.v[c].n, sizeof(out[c].n));
        out[c].delta = L.v[c].delta;
        memset(out[c].P, 0, sizeof(out[c].P));
    }
    free(L.v);
    return 0;
}

/* Contacts of selected particles only (brute force against all N, walls and plates): the
 * full-size sampled check of the pair set.  Same predicate and orientation as detect_all. */
int32_t or_contacts_of(const or_world *w, const int64_t *idx, int64_t nidx, or_contact *out, int64_t cap,
                       int64_t *n_out)
{
    raw_list L = {0, 0, 0};
    const int64_t N = w->n;
    for (int64_t q = 0; q < nidx; q++) {
        const int64_t i = idx[q];
        for (int64_t j = 0; j < N; j++) {
            if (j == i) continue;
            int64_t a = i, b = j;
            if (w->gid[j] < w->gid[i]) { a = j; b = i; }
            double dx = w->x[3 * b + 0] - w->x[3 * a + 0];
            double dy = w->x[3 * b + 1] - w->x[3 * a + 1];
            double dz = w->x[3 * b + 2] - w->x[3 * a + 2];
            double d2 = (dx * dx + dy * dy) + dz * dz;
            double R = w->r[a] + w->r[b];
            if (!(d2 < R * R) || d2 == 0.0) continue;
            double d = sqrt(d2);
            raw_contact c;
            c.key = ((uint64_t)w->gid[a] << 32) | (uint64_t)w->gid[b];
            c.a = a; c.b = b; c.kind = 0; c.idx = -1;
            c.n[0] = dx / d; c.n[1] = dy / d; c.n[2] = dz / d;
            c.delta = R - d;
            if (push(&L, &c)) { free(L.v); return -1; }
        }
        for (int32_t k = 0; k < w->n_walls; k++) {
            const or_wall *W = &w->walls[k];
            double s = ((w->x[3 * i] - W->p[0]) * W->n[0] + (w->x[3 * i + 1] - W->p[1]) * W->n[1])
                       + (w->x[3 * i + 2] - W->p[2]) * W->n[2];
            if (!(s < w->r[i])) continue;
            raw_contact c;
            c.key = ((uint64_t)w->gid[i] << 32) | (uint64_t)WALL_KEY(W->id);
            c.a = i; c.b = -1; c.kind = 1; c.idx = k;
            c.n[0] = -W->n[0]; c.n[1] = -W->n[1]; c.n[2] = -W->n[2];
            c.delta = w->r[i] - s;
            if (push(&L, &c)) { free(L.v); return -1; }
        }
    }
    qsort(L.v, (size_t)L.n, sizeof(raw_contact), cmp_raw);
    int64_t m = 0;
    for (int64_t c = 0; c < L.n; c++) {
        if (m && L.v[c].key == out[m - 1].key) continue;       /* pair found from both ends */
        if (m >= cap) { free(L.v); return -1; }
        out[m].key = L.v[c].key;
        memcpy(out[m].n, L.v[c].n, sizeof(out[m].n));
        out[m].delta = L.v[c].delta;
        memset(out[m].P, 0, sizeof(out[m].P));
        m++;
    }
    *n_out = m;
    free(L.v);
    return 0;
}

/* ---------------------------------------------------------------- the step */
typedef struct {
    raw_contact g;
    double Rs;          /* R* = r_a r_b/(r_a+r_b); r for walls and plates (reading R7) */
    double kn;          /* k_n = E* sqrt(d*)/3, or k_lin */
    double la[3], lb[3];/* lever arms a->contact point, b->contact point (reading R10) */
    double mu_t, mu_r;
    double S, bias;     /* SPOOK row: Sigma-hat and b (P-units) */
    double P[7];
    double dP[7];
    double inc[9];      /* this sweep's increments: dL = dPn n + dPt, l_a x dPt + dPr, l_b x dPt + dPr */
    double un_minus;    /* n.(v_b - v_a) at the start of the step */
    int impacting;
} row;

static int cmp_key_hist(const void *x, const void *y)
{
    uint64_t a = ((const or_contact *)x)->key, b = ((const or_contact *)y)->key;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* velocity of body b of a contact (particle, moving wall, or translating plate) */
static void body_b_vel(const or_world *w, const row *R, const double *v, const double *om,
                       double *vb, double *wb)
{
    if (R->g.kind == 0) {
        for (int k = 0; k < 3; k++) { vb[k] = v[3 * R->g.b + k]; wb[k] = om[3 * R->g.b + k]; }
    } else if (R->g.kind == 1) {
        const or_wall *W = &w->walls[R->g.idx];
        for (int k = 0; k < 3; k++) { vb[k] = W->vel * W->n[k]; wb[k] = 0.0; }
    } else {
        const or_plate *P = &w->plates[R->g.idx];
        for (int k = 0; k < 3; k++) { vb[k] = P->vel[k]; wb[k] = 0.0; }
    }
}

/*
 * One Jacobi sweep (P:134 solver, P:115-125 laws; Jacobi with mass splitting, reading R2):
 * every contact is solved from the sweep-start velocities (v, om) with the split inverse
 * masses wa = c_a/m_a, wta = c_a/I_a, in the contact-local order normal -> friction ->
 * rolling, and the impulse increments are summed per body with the real masses.
 */
static void sweep(const or_world *w, const or_params *p, row *R, int64_t nc,
                  const int32_t *cnt, const double *minv, const double *Iinv,
                  double *v, double *om, const int64_t *inc_s, const int64_t *inc_l, double *accP)
{
    if (accP) memset(accP, 0, sizeof(double) * 3 * (size_t)w->n_plates);
    const int64_t N = w->n;
    /* every contact from the sweep-start velocities (order-free: OpenMP over contacts) */
#pragma omp parallel for schedule(static) if (nc > 4096)
    for (int64_t c = 0; c < nc; c++) {
        row *r = &R[c];
        const int64_t a = r->g.a;
        const double *n = r->g.n;
        double va[3], wa_[3], vb[3], wb_[3];
        for (int k = 0; k < 3; k++) { va[k] = v[3 * a + k]; wa_[k] = om[3 * a + k]; }
        body_b_vel(w, r, v, om, vb, wb_);
        const double wA = cnt[a] * minv[a], wtA = cnt[a] * Iinv[a];
        double wB = 0.0, wtB = 0.0;
        if (r->g.kind == 0) { wB = cnt[r->g.b] * minv[r->g.b]; wtB = cnt[r->g.b] * Iinv[r->g.b]; }
        const double Dn = wA + wB;
        const double Dt = wA + wB + dot3(r->la, r->la) * wtA + dot3(r->lb, r->lb) * wtB;
        const double Dr = wtA + wtB;

        /* 1. normal row: P_n' = max(0, P_n - (u_n + S P_n - b)/(D_n + S)) */
        double dv[3];
        for (int k = 0; k < 3; k++) dv[k] = vb[k] - va[k];
        double un = dot3(n, dv);
        double Pn0 = r->P[0];
        double Pn = Pn0 - (un + r->S * Pn0 - r->bias) / (Dn + r->S);
        if (Pn < 0.0) Pn = 0.0;
        double dPn = Pn - Pn0;
        for (int k = 0; k < 3; k++) { va[k] -= wA * dPn * n[k]; vb[k] += wB * dPn * n[k]; }

        /* 2. friction: u = (v_b + w_b x l_b) - (v_a + w_a x l_a), tangential part, disc of
         *    radius mu_t P_n' (maximum dissipation P:123-125) */
        double ca[3], cb[3], u[3], ut[3];
        cross3(wa_, r->la, ca);
        cross3(wb_, r->lb, cb);
        for (int k = 0; k < 3; k++) u[k] = (vb[k] + cb[k]) - (va[k] + ca[k]);
        double uu = dot3(u, n);
        for (int k = 0; k < 3; k++) ut[k] = u[k] - uu * n[k];
        double Pt[3];
        for (int k = 0; k < 3; k++) Pt[k] = r->P[1 + k] - ut[k] / Dt;
        double lim = r->mu_t * Pn, mag = norm3(Pt);
        if (mag > lim) { double s = mag > 0.0 ? lim / mag : 0.0; for (int k = 0; k < 3; k++) Pt[k] *= s; }
        double dPt[3];
        for (int k = 0; k < 3; k++) dPt[k] = Pt[k] - r->P[1 + k];
        double ta[3], tb[3];
        cross3(r->la, dPt, ta);
        cross3(r->lb, dPt, tb);
        for (int k = 0; k < 3; k++) {
            va[k] -= wA * dPt[k];
            wa_[k] -= wtA * ta[k];
            vb[k] += wB * dPt[k];
            wb_[k] += wtB * tb[k];
        }

        /* 3. rolling: u_r = w_b - w_a, ball of radius mu_r R* P_n' (R7/R8) */
        double ur[3];
        for (int k = 0; k < 3; k++) ur[k] = wb_[k] - wa_[k];
        if (p->rolling_dims == 2) { double q = dot3(ur, n); for (int k = 0; k < 3; k++) ur[k] -= q * n[k]; }
        double Pr[3];
        for (int k = 0; k < 3; k++) Pr[k] = r->P[4 + k] - ur[k] / Dr;
        lim = r->mu_r * r->Rs * Pn;
        mag = norm3(Pr);
        if (mag > lim) { double s = mag > 0.0 ? lim / mag : 0.0; for (int k = 0; k < 3; k++) Pr[k] *= s; }
        double dPr[3];
        for (int k = 0; k < 3; k++) dPr[k] = Pr[k] - r->P[4 + k];

        /* 4. increments: a gets -(dPn n + dPt), -(l_a x dPt + dPr); b the opposite sign with
         *    its own lever arm (summed per body below) */
        for (int k = 0; k < 3; k++) {
            r->inc[k] = dPn * n[k] + dPt[k];
            r->inc[3 + k] = ta[k] + dPr[k];
            r->inc[6 + k] = tb[k] + dPr[k];
        }
        r->P[0] = Pn;
        for (int k = 0; k < 3; k++) { r->P[1 + k] = Pt[k]; r->P[4 + k] = Pr[k]; }
    }
    /* monolithic plate (R18b): the plate receives +(dPn n + dPt) */
    if (accP)
        for (int64_t c = 0; c < nc; c++)
            if (R[c].g.kind == 2) for (int k = 0; k < 3; k++) accP[3 * R[c].g.idx + k] += R[c].inc[k];
    /* 5. body update with the real masses (= mass-splitting average): per body, its contacts'
     *    increments in contact order (inc_s/inc_l lists them by increasing contact index) */
#pragma omp parallel for schedule(static) if (N > 4096)
    for (int64_t i = 0; i < N; i++) {
        double aL[3] = {0.0, 0.0, 0.0}, aA[3] = {0.0, 0.0, 0.0};
        for (int64_t t = inc_s[i]; t < inc_s[i + 1]; t++) {
            const row *r = &R[inc_l[t] >> 1];
            if (inc_l[t] & 1) for (int k = 0; k < 3; k++) { aL[k] += r->inc[k]; aA[k] += r->inc[6 + k]; }
            else for (int k = 0; k < 3; k++) { aL[k] -= r->inc[k]; aA[k] -= r->inc[3 + k]; }
        }
        for (int k = 0; k < 3; k++) {
            v[3 * i + k] += minv[i] * aL[k];
            om[3 * i + k] += Iinv[i] * aA[k];
        }
    }
}

/* ---------------------------------------------------------------- coloured Gauss-Seidel (NEXT-1)
 * The paper solves the MCP with projected Gauss-Seidel: contacts one after the other,
 * each from the latest velocities, its impulse increment applied at once with the real masses.
 * The order used here: by colour of a greedy colouring of the contact conflict graph (two
 * contacts conflict if they share a particle), then by key.  Contacts of one colour touch
 * disjoint particles, so within a colour the order does not matter. */
uint64_t or_splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

static const uint64_t *g_pri_key;      /* qsort context (single-threaded oracle) */
static const uint64_t *g_pri;
static int cmp_priority(const void *x, const void *y)
{
    const int64_t i = *(const int64_t *)x, j = *(const int64_t *)y;
    if (g_pri[i] != g_pri[j]) return g_pri[i] > g_pri[j] ? -1 : 1;       /* decreasing priority */
    return g_pri_key[i] < g_pri_key[j] ? -1 : (g_pri_key[i] > g_pri_key[j] ? 1 : 0);
}

int32_t or_color_contacts(int64_t nc, const uint64_t *key, const int64_t *a, const int64_t *b, int64_t n_particles,
                          int32_t *color)
{
    uint64_t *pri = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nc ? nc : 1));
    int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nc ? nc : 1));
    uint64_t *used = (uint64_t *)calloc((size_t)(n_particles ? n_particles : 1) * 4, sizeof(uint64_t));
    int32_t ncol = 0;
    for (int64_t c = 0; c < nc; c++) { pri[c] = or_splitmix64(key[c]); ord[c] = c; color[c] = -1; }
    g_pri = pri;
    g_pri_key = key;
    qsort(ord, (size_t)nc, sizeof(int64_t), cmp_priority);
    for (int64_t t = 0; t < nc; t++) {
        const int64_t c = ord[t];
        int32_t col = -1;
        for (int q = 0; q < 256 && col < 0; q++) {
            const uint64_t bit = 1ULL << (q & 63);
            const int wa = (used[4 * a[c] + (q >> 6)] & bit) != 0;
            const int wb = b[c] >= 0 ? (used[4 * b[c] + (q >> 6)] & bit) != 0 : 0;
            if (!wa && !wb) col = q;
        }
        if (col < 0) { ncol = -1; break; }
        color[c] = col;
        used[4 * a[c] + (col >> 6)] |= 1ULL << (col & 63);
        if (b[c] >= 0) used[4 * b[c] + (col >> 6)] |= 1ULL << (col & 63);
        if (col + 1 > ncol) ncol = col + 1;
    }
    free(pri); free(ord); free(used);
    return ncol;
}

/* One projected Gauss-Seidel sweep in the given contact order: the same contact-local update as
 * the Jacobi sweep (normal -> friction -> rolling) with the real inverse masses, its increments
 * applied to the bodies immediately. */
static void sweep_gs(const or_world *w, const or_params *p, row *R, int64_t nc, const int64_t *order,
                     const double *minv, const double *Iinv, double *v, double *om)
{
    for (int64_t t = 0; t < nc; t++) {
        row *r = &R[order[t]];
        const int64_t a = r->g.a;
        const double *n = r->g.n;
        double va[3], wa_[3], vb[3], wb_[3];
        for (int k = 0; k < 3; k++) { va[k] = v[3 * a + k]; wa_[k] = om[3 * a + k]; }
        body_b_vel(w, r, v, om, vb, wb_);
        const double wA = minv[a], wtA = Iinv[a];
        double wB = 0.0, wtB = 0.0;
        if (r->g.kind == 0) { wB = minv[r->g.b]; wtB = Iinv[r->g.b]; }
        const double Dn = wA + wB;
        const double Dt = wA + wB + dot3(r->la, r->la) * wtA + dot3(r->lb, r->lb) * wtB;
        const double Dr = wtA + wtB;
        double dv[3];
        for (int k = 0; k < 3; k++) dv[k] = vb[k] - va[k];
        const double Pn0 = r->P[0];
        double Pn = Pn0 - (dot3(n, dv) + r->S * Pn0 - r->bias) / (Dn + r->S);
        if (Pn < 0.0) Pn = 0.0;
        const double dPn = Pn - Pn0;
        for (int k = 0; k < 3; k++) { va[k] -= wA * dPn * n[k]; vb[k] += wB * dPn * n[k]; }
        double ca[3], cb[3], u[3], ut[3];
        cross3(wa_, r->la, ca);
        cross3(wb_, r->lb, cb);
        for (int k = 0; k < 3; k++) u[k] = (vb[k] + cb[k]) - (va[k] + ca[k]);
        const double uu = dot3(u, n);
        for (int k = 0; k < 3; k++) ut[k] = u[k] - uu * n[k];
        double Pt[3];
        for (int k = 0; k < 3; k++) Pt[k] = r->P[1 + k] - ut[k] / Dt;
        double lim = r->mu_t * Pn, mag = norm3(Pt);
        if (mag > lim) { double s = mag > 0.0 ? lim / mag : 0.0; for (int k = 0; k < 3; k++) Pt[k] *= s; }
        double dPt[3], ta[3], tb[3];
        for (int k = 0; k < 3; k++) dPt[k] = Pt[k] - r->P[1 + k];
        cross3(r->la, dPt, ta);
        cross3(r->lb, dPt, tb);
        for (int k = 0; k < 3; k++) {
            va[k] -= wA * dPt[k];
            wa_[k] -= wtA * ta[k];
            vb[k] += wB * dPt[k];
            wb_[k] += wtB * tb[k];
        }
        double ur[3];
        for (int k = 0; k < 3; k++) ur[k] = wb_[k] - wa_[k];
        if (p->rolling_dims == 2) { double q = dot3(ur, n); for (int k = 0; k < 3; k++) ur[k] -= q * n[k]; }
        double Pr[3];
        for (int k = 0; k < 3; k++) Pr[k] = r->P[4 + k] - ur[k] / Dr;
        lim = r->mu_r * r->Rs * Pn;
        mag = norm3(Pr);
        if (mag > lim) { double s = mag > 0.0 ? lim / mag : 0.0; for (int k = 0; k < 3; k++) Pr[k] *= s; }
        double dPr[3];
        for (int k = 0; k < 3; k++) dPr[k] = Pr[k] - r->P[4 + k];
        /* Gauss-Seidel: the increments go to the bodies now */
        for (int k = 0; k < 3; k++) {
            v[3 * a + k] -= minv[a] * (dPn * n[k] + dPt[k]);
            om[3 * a + k] -= Iinv[a] * (ta[k] + dPr[k]);
        }
        if (r->g.kind == 0) {
            const int64_t b = r->g.b;
            for (int k = 0; k < 3; k++) {
                v[3 * b + k] += minv[b] * (dPn * n[k] + dPt[k]);
                om[3 * b + k] += Iinv[b] * (tb[k] + dPr[k]);
            }
        }
        r->P[0] = Pn;
        for (int k = 0; k < 3; k++) { r->P[1 + k] = Pt[k]; r->P[4 + k] = Pr[k]; }
    }
}

/* contact order of the Gauss-Seidel sweeps: by colour, then by key (rows are in key order) */
static int32_t gs_order(const row *R, int64_t nc, int64_t N, int64_t *order)
{
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nc ? nc : 1));
    int64_t *a = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nc ? nc : 1));
    int64_t *b = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nc ? nc : 1));
    int32_t *col = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nc ? nc : 1));
    for (int64_t c = 0; c < nc; c++) { key[c] = R[c].g.key; a[c] = R[c].g.a; b[c] = R[c].g.kind == 0 ? R[c].g.b : -1; }
    const int32_t ncol = or_color_contacts(nc, key, a, b, N, col);
    int64_t t = 0;
    for (int32_t q = 0; q < ncol; q++)
        for (int64_t c = 0; c < nc; c++)
            if (col[c] == q) order[t++] = c;
    free(key); free(a); free(b); free(col);
    return ncol;
}

/* apply impulses P of every row to the bodies with real masses (warm start) */
static void apply_impulses(const or_world *w, row *R, int64_t nc, const double *minv,
                           const double *Iinv, double *v, double *om)
{
    for (int64_t c = 0; c < nc; c++) {
        const row *r = &R[c];
        double L[3], ta[3], tb[3];
        for (int k = 0; k < 3; k++) L[k] = r->P[0] * r->g.n[k] + r->P[1 + k];
        cross3(r->la, &r->P[1], ta);
        cross3(r->lb, &r->P[1], tb);
        const int64_t a = r->g.a;
        for (int k = 0; k < 3; k++) {
            v[3 * a + k] -= minv[a] * L[k];
            om[3 * a + k] -= Iinv[a] * (ta[k] + r->P[4 + k]);
        }
        if (r->g.kind == 0) {
            const int64_t b = r->g.b;
            for (int k = 0; k < 3; k++) {
                v[3 * b + k] += minv[b] * L[k];
                om[3 * b + k] += Iinv[b] * (tb[k] + r->P[4 + k]);
            }
        }
    }
    (void)w;
}

static void clamp_cones(row *r, int rolling_dims)
{
    /* warm start: re-project P_t onto the current tangent plane, clamp to the cones (R12) */
    const double *n = r->g.n;
    double q = dot3(&r->P[1], n);
    for (int k = 0; k < 3; k++) r->P[1 + k] -= q * n[k];
    if (rolling_dims == 2) { q = dot3(&r->P[4], n); for (int k = 0; k < 3; k++) r->P[4 + k] -= q * n[k]; }
    if (r->P[0] < 0.0) r->P[0] = 0.0;
    double lim = r->mu_t * r->P[0], mag = norm3(&r->P[1]);
    if (mag > lim) { double s = mag > 0.0 ? lim / mag : 0.0; for (int k = 0; k < 3; k++) r->P[1 + k] *= s; }
    lim = r->mu_r * r->Rs * r->P[0];
    mag = norm3(&r->P[4]);
    if (mag > lim) { double s = mag > 0.0 ? lim / mag : 0.0; for (int k = 0; k < 3; k++) r->P[4 + k] *= s; }
}

int32_t or_step(or_world *w, const or_params *p, const or_contact *hist, int64_t n_hist,
                or_contact *out, int64_t cap, int64_t *n_out, double *F, double *T,
                or_report *rep)
{
    const int64_t N = w->n;
    const double h = p->h;
    const double gnorm = sqrt(dot3(p->g, p->g));
    const double v_imp = p->v_imp < 0.0 ? 20.0 * gnorm * h : p->v_imp;
    const int32_t n_imp = p->n_imp > 0 ? p->n_imp : p->n_it;
    const double Ups = 1.0 / (1.0 + 4.0 * p->damp_steps);  /* 1/(1+4 tau/h), tau = damp*h */
    const double Es = 1.0 / (2.0 * (1.0 - p->nu * p->nu) / p->E);  /* identical materials (R17) */
    int32_t rc = 0;
    memset(rep, 0, sizeof(*rep));

    /* 1. detection */
    raw_list L = {0, 0, 0};
    int64_t n_degen = 0;
    if (detect_all(w, &L, &n_degen)) { free(L.v); return -1; }
    const int64_t nc = L.n;
    *n_out = nc;
    if (nc > cap) { free(L.v); return -1; }

    double *minv = (double *)malloc(sizeof(double) * (size_t)(N ? N : 1));
    double *Iinv = (double *)malloc(sizeof(double) * (size_t)(N ? N : 1));
    int32_t *cnt = (int32_t *)calloc((size_t)(N ? N : 1), sizeof(int32_t));
    int64_t *inc_s = (int64_t *)calloc((size_t)N + 2, sizeof(int64_t));
    int64_t *inc_l = (int64_t *)malloc(sizeof(int64_t) * (2 * (size_t)nc + 1));
    row *R = (row *)calloc((size_t)(nc ? nc : 1), sizeof(row));
    or_contact *H = NULL;
    for (int64_t i = 0; i < N; i++) {
        double m, I;
        or_mass_inertia(2.0 * w->r[i], p->rho, &m, &I);
        minv[i] = 1.0 / m;
        Iinv[i] = 1.0 / I;
    }

    /* 2. contact constants (reading R7, R10, R17) */
    for (int64_t c = 0; c < nc; c++) {
        row *r = &R[c];
        r->g = L.v[c];
        const double ra = w->r[r->g.a];
        const double *n = r->g.n;
        double ds;
        if (r->g.kind == 0) {
            const double rb = w->r[r->g.b];
            r->Rs = ra * rb / (ra + rb);
            ds = 2.0 * r->Rs;                       /* d* = (1/d_a + 1/d_b)^-1 */
            for (int k = 0; k < 3; k++) r->lb[k] = -(rb - 0.5 * r->g.delta) * n[k];
            r->mu_t = p->mu_t; r->mu_r = p->mu_r;
        } else {
            r->Rs = ra;
            ds = 2.0 * ra;                          /* flat tool: d* = d */
            for (int k = 0; k < 3; k++) r->lb[k] = 0.0;
            if (r->g.kind == 1) { r->mu_t = w->walls[r->g.idx].mu_t; r->mu_r = w->walls[r->g.idx].mu_r; }
            else { r->mu_t = w->plates[r->g.idx].mu_t; r->mu_r = w->plates[r->g.idx].mu_r; }
        }
        for (int k = 0; k < 3; k++) r->la[k] = (ra - 0.5 * r->g.delta) * n[k];
        r->kn = (p->e_H == 1.0) ? p->k_lin : Es * sqrt(ds) / 3.0;
        cnt[r->g.a]++;
        if (r->g.kind == 0) cnt[r->g.b]++;
        if (r->g.kind == 0) rep->n_pp++; else if (r->g.kind == 1) rep->n_wall++; else rep->n_plate++;
    }
    rep->n_contacts = nc;
    rep->n_degenerate = n_degen;
    /* per body, its contacts in increasing contact index (entry = c << 1 | is-body-b): the order
     * in which the sweep adds a body's increments */
    for (int64_t i = 0; i < N; i++) inc_s[i + 1] = inc_s[i] + cnt[i];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N ? N : 1));
        for (int64_t i = 0; i < N; i++) fill[i] = inc_s[i];
        for (int64_t c = 0; c < nc; c++) {
            inc_l[fill[R[c].g.a]++] = c << 1;
            if (R[c].g.kind == 0) inc_l[fill[R[c].g.b]++] = (c << 1) | 1;
        }
        free(fill);
    }
    const int gs = p->ordering == 1;
    int64_t *order = NULL;
    if (gs) {
        order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nc ? nc : 1));
        if (gs_order(R, nc, N, order) < 0) {                    /* more than 256 colours */
            free(L.v); free(minv); free(Iinv); free(cnt); free(inc_s); free(inc_l); free(R); free(order);
            return -3;
        }
    }

    /* 3. impact trigger: u_n^- = n.(v_b^k - v_a^k) < -v_imp */
    int fired = 0;
    for (int64_t c = 0; c < nc; c++) {
        row *r = &R[c];
        double vb[3], wb[3], dv[3];
        body_b_vel(w, r, w->v, w->w, vb, wb);
        for (int k = 0; k < 3; k++) dv[k] = vb[k] - w->v[3 * r->g.a + k];
        r->un_minus = dot3(r->g.n, dv);
        r->impacting = r->un_minus < -v_imp;
        if (r->impacting) fired = 1;
    }
    rep->impact_fired = fired;
    if (fired) {
        /* impact stage: from P = 0, Sigma = 0, b = -e u_n^- on impacting normals, 0 elsewhere;
         * friction and rolling cones active; applied to v^k, impulses discarded (R13) */
        for (int64_t c = 0; c < nc; c++) {
            row *r = &R[c];
            memset(r->P, 0, sizeof(r->P));
            r->S = 0.0;
            r->bias = r->impacting ? -p->e_rest * r->un_minus : 0.0;
        }
        /* monolithic plates (R18b): force-driven axes take their contacts' impact impulses too */
        const int mono_i = p->plate_coupling == 1 && !gs && w->n_plates > 0;
        double *accPi = mono_i ? (double *)calloc(3 * (size_t)w->n_plates, sizeof(double)) : NULL;
        for (int32_t s = 0; s < n_imp; s++) {
            if (gs) sweep_gs(w, p, R, nc, order, minv, Iinv, w->v, w->w);
            else sweep(w, p, R, nc, cnt, minv, Iinv, w->v, w->w, inc_s, inc_l, accPi);
            if (mono_i)
                for (int32_t q = 0; q < w->n_plates; q++) {
                    or_plate *P = &w->plates[q];
                    for (int k = 0; k < 3; k++)
                        if (P->mode[k] == 2) P->vel[k] += accPi[3 * q + k] / P->mass;
                }
        }
        free(accPi);
    }

    /* 4. main-stage rows (SPOOK; reading R4):
     *    S = 4 Ups / (h^2 e_H k_n delta^(2 e_H - 2)),  b = (4 Ups/h)(delta/e_H) + Ups n.(v_b^k - v_a^k) */
    for (int64_t c = 0; c < nc; c++) {
        row *r = &R[c];
        double vb[3], wb[3], dv[3];
        body_b_vel(w, r, w->v, w->w, vb, wb);
        for (int k = 0; k < 3; k++) dv[k] = vb[k] - w->v[3 * r->g.a + k];
        const double un = dot3(r->g.n, dv);
        const double dl = r->g.delta;
        r->S = 4.0 * Ups / (h * h * p->e_H * r->kn * pow(dl, 2.0 * p->e_H - 2.0));
        r->bias = (4.0 * Ups / h) * (dl / p->e_H) + Ups * un;
    }

    /* 5. warm start from the history: same key -> previous impulses */
    if (n_hist > 0) {
        H = (or_contact *)malloc(sizeof(or_contact) * (size_t)n_hist);
        memcpy(H, hist, sizeof(or_contact) * (size_t)n_hist);
        qsort(H, (size_t)n_hist, sizeof(or_contact), cmp_key_hist);
    }
    for (int64_t c = 0; c < nc; c++) {
        row *r = &R[c];
        memset(r->P, 0, sizeof(r->P));
        if (H) {
            or_contact probe;
            probe.key = r->g.key;
            const or_contact *f = (const or_contact *)bsearch(&probe, H, (size_t)n_hist, sizeof(or_contact), cmp_key_hist);
            if (f) { memcpy(r->P, f->P, sizeof(r->P)); clamp_cones(r, p->rolling_dims); }
        }
    }

    /* 6. external force: v* = v^k + h g, then v(0) = v* + M^-1 sum J^T P_hist */
    for (int64_t i = 0; i < N; i++)
        for (int k = 0; k < 3; k++) w->v[3 * i + k] += h * p->g[k];
    apply_impulses(w, R, nc, minv, Iinv, w->v, w->w);

    /* 6b. monolithic plates (R18b): a force-driven axis is a body of this solve -- it takes the
     *     external impulse h F and the warm-start impulses of its contacts, V += (h F + sum L)/M,
     *     and after every sweep the increments of its contacts, V += sum dL / M (Jacobi with the
     *     real mass = the mass-splitting average over its contacts); likewise in the impact stage.
     *     In the contact rows the plate keeps an infinite mass (the diagonal only sets the step
     *     of the projected iteration; the fixed point is the coupled MCP's) */
    const int mono = p->plate_coupling == 1 && !gs && w->n_plates > 0;
    double *accP = mono ? (double *)calloc(3 * (size_t)w->n_plates, sizeof(double)) : NULL;
    if (mono) {
        for (int64_t c = 0; c < nc; c++) {
            row *r = &R[c];
            if (r->g.kind != 2) continue;
            for (int k = 0; k < 3; k++) accP[3 * r->g.idx + k] += r->P[0] * r->g.n[k] + r->P[1 + k];
        }
        for (int32_t q = 0; q < w->n_plates; q++) {
            or_plate *P = &w->plates[q];
            for (int k = 0; k < 3; k++)
                if (P->mode[k] == 2) P->vel[k] += (h * P->target[k] + accP[3 * q + k]) / P->mass;
        }
    }

    /* 7. N_it sweeps: Jacobi, or coloured Gauss-Seidel */
    for (int32_t s = 0; s < p->n_it; s++) {
        if (gs) sweep_gs(w, p, R, nc, order, minv, Iinv, w->v, w->w);
        else sweep(w, p, R, nc, cnt, minv, Iinv, w->v, w->w, inc_s, inc_l, accP);
        if (mono)
            for (int32_t q = 0; q < w->n_plates; q++) {
                or_plate *P = &w->plates[q];
                for (int k = 0; k < 3; k++)
                    if (P->mode[k] == 2) P->vel[k] += accP[3 * q + k] / P->mass;
            }
    }
    free(accP);

    /* 8. outputs: forces/torques (P/h sums), plate reactions, residuals (O6, O9) */
    if (F) memset(F, 0, sizeof(double) * 3 * (size_t)N);
    if (T) memset(T, 0, sizeof(double) * 3 * (size_t)N);
    for (int32_t q = 0; q < w->n_plates; q++) for (int k = 0; k < 3; k++) w->plates[q].force[k] = 0.0;
    for (int64_t c = 0; c < nc; c++) {
        row *r = &R[c];
        double Lc[3], ta[3], tb[3];
        for (int k = 0; k < 3; k++) Lc[k] = r->P[0] * r->g.n[k] + r->P[1 + k];
        cross3(r->la, &r->P[1], ta);
        cross3(r->lb, &r->P[1], tb);
        const int64_t a = r->g.a;
        if (F) for (int k = 0; k < 3; k++) F[3 * a + k] -= Lc[k] / h;
        if (T) for (int k = 0; k < 3; k++) T[3 * a + k] -= (ta[k] + r->P[4 + k]) / h;
        if (r->g.kind == 0) {
            const int64_t b = r->g.b;
            if (F) for (int k = 0; k < 3; k++) F[3 * b + k] += Lc[k] / h;
            if (T) for (int k = 0; k < 3; k++) T[3 * b + k] += (tb[k] + r->P[4 + k]) / h;
        } else if (r->g.kind == 2) {
            for (int k = 0; k < 3; k++) w->plates[r->g.idx].force[k] += Lc[k] / h;
        }
        /* residuals at the final velocities */
        double vb[3], wb[3], dv[3];
        body_b_vel(w, r, w->v, w->w, vb, wb);
        for (int k = 0; k < 3; k++) dv[k] = vb[k] - w->v[3 * a + k];
        double wn = dot3(r->g.n, dv) + r->S * r->P[0] - r->bias;
        double res = fabs(r->P[0] < wn ? r->P[0] : wn);
        if (res > rep->max_normal_residual) rep->max_normal_residual = res;
        double e1 = norm3(&r->P[1]) - r->mu_t * r->P[0];
        double e2 = norm3(&r->P[4]) - r->mu_r * r->Rs * r->P[0];
        if (e1 > rep->max_cone_excess) rep->max_cone_excess = e1;
        if (e2 > rep->max_cone_excess) rep->max_cone_excess = e2;
    }

    /* 9. integrate: x^{k+1} = x^k + h v^{k+1}; walls and plates move with the velocity
     *    used in this step, then drives update plate velocities for the next step (R18) */
    int bad = 0;
    double ke = 0.0, maxv = 0.0;
    for (int64_t i = 0; i < N; i++) {
        for (int k = 0; k < 3; k++) w->x[3 * i + k] += h * w->v[3 * i + k];
        double m = 1.0 / minv[i], I = 1.0 / Iinv[i];
        double v2 = dot3(&w->v[3 * i], &w->v[3 * i]), w2 = dot3(&w->w[3 * i], &w->w[3 * i]);
        ke += 0.5 * m * v2 + 0.5 * I * w2;
        if (sqrt(v2) > maxv) maxv = sqrt(v2);
        for (int k = 0; k < 3; k++)
            if (!isfinite(w->x[3 * i + k]) || !isfinite(w->v[3 * i + k]) || !isfinite(w->w[3 * i + k])) bad = 1;
    }
    for (int32_t k = 0; k < w->n_walls; k++) {
        or_wall *W = &w->walls[k];
        for (int j = 0; j < 3; j++) W->p[j] += h * W->vel * W->n[j];
    }
    const double t1 = w->time + h;
    for (int32_t q = 0; q < w->n_plates; q++) {
        or_plate *P = &w->plates[q];
        for (int k = 0; k < 3; k++) P->pos[k] += h * P->vel[k];
        for (int k = 0; k < 3; k++) {
            if (P->mode[k] == 2) {
                /* staggered force axis (R18); monolithic (R18b): the solve set V already */
                if (p->plate_coupling != 1 || gs) P->vel[k] += h * (P->target[k] + P->force[k]) / P->mass;
                P->motor[k] = P->target[k];
                continue;
            }
            /* locked (u = 0) or motor G_j v = u_j(t) with u ramped over ramp[k] */
            double u = 0.0;
            if (P->mode[k] == 1) {
                double s = P->ramp[k] > 0.0 ? (t1 - P->t0[k]) / P->ramp[k] : 1.0;
                if (s > 1.0) s = 1.0;
                if (s < 0.0) s = 0.0;
                u = P->target[k] * s;
            }
            /* staggered motor (R18): the force reaching u at t1 against this step's contact
             * reaction; Eq. 4 limits lambda_min <= lambda <= lambda_max on velocity axes */
            double lambda = P->mass * (u - P->vel[k]) / h - P->force[k];
            if (P->mode[k] == 1 && P->limit[k] && (lambda < P->fmin[k] || lambda > P->fmax[k])) {
                lambda = lambda < P->fmin[k] ? P->fmin[k] : P->fmax[k];
                P->vel[k] += h * (lambda + P->force[k]) / P->mass;
            } else {
                P->vel[k] = u;
            }
            P->motor[k] = lambda;
        }
    }
    w->time = t1;
    rep->ke = ke;
    rep->max_v = maxv;

    /* 10. history out, sorted by key (= contact order) */
    for (int64_t c = 0; c < nc; c++) {
        out[c].key = R[c].g.key;
        memcpy(out[c].n, R[c].g.n, sizeof(out[c].n));
        out[c].delta = R[c].g.delta;
        memcpy(out[c].P, R[c].P, sizeof(out[c].P));
        for (int k = 0; k < 7; k++) if (!isfinite(R[c].P[k])) bad = 1;
    }
    if (bad) rc = -2;
    free(L.v); free(minv); free(Iinv); free(cnt); free(inc_s); free(inc_l); free(R); free(H); free(order);
    return rc;
}
