/*
 * oracle.h -- fp64 CPU oracle for one nonsmooth-DEM time step (TEST INFRASTRUCTURE ONLY).
 *
 * This header and dem_oracle.c are the plain, slow, obviously-correct reference the CUDA
 * path is checked against.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs may load liboracle.so.  It shares no code, header, table or constant
 * generator with paper_2501_05300_b200/ (the product); the two are independent by design.
 *
 * Paper: Pogulis & Servin, "Local particle refinement in terramechanical simulations"
 * (arXiv 2501.05300), /root/reference/PAPER.md.  Citations "P:n" are PAPER.md lines, "S:n"
 * SPEC.md lines; readings of silent/garbled passages are listed in DESIGN.md §3 ("R#").
 *
 * Units are SI throughout; z is up; gravity is a parameter.
 */
#ifndef DEM_ORACLE_H
#define DEM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Material + solver parameters (P:157 material, P:127-129 contact law, P:132-138 solver). */
typedef struct {
    double rho, E, nu;        /* particle density, Young's modulus, Poisson ratio */
    double mu_t, mu_r;        /* inter-particle Coulomb and rolling coefficients */
    double e_rest;            /* Newton restitution for the impact stage */
    double h;                 /* time step dt */
    int32_t n_it;             /* main-stage sweeps */
    int32_t n_imp;            /* impact-stage sweeps (<=0 -> n_it) */
    double e_H;               /* Hertz exponent: 1.25, or 1.0 = linear model */
    double k_lin;             /* linear stiffness [N/m], used iff e_H == 1 (reading R3) */
    double damp_steps;        /* SPOOK damping time tau = damp_steps*h (4.5) */
    double v_imp;             /* impact threshold; <0 -> 20|g|h; >=1e30 disables */
    double g[3];              /* gravity */
    int32_t rolling_dims;     /* 3 (default) or 2 (rolling row projected on tangent plane) */
    int32_t ordering;         /* 0: Jacobi with mass splitting (reading R2); 1: coloured projected
                                 Gauss-Seidel (P:134 PGS), see or_color_contacts */
    int32_t plate_coupling;   /* force-driven plate axes: 0 staggered after the solve (reading R18);
                                 1 monolithic: the plate is a body of the main-stage solve (reading
                                 R18b; Jacobi ordering only) */
    int32_t pad;
} or_params;

/* Static or kinematic plane wall: contact iff (X-p).n < r (reading R17). */
typedef struct {
    double p[3];              /* a point of the plane */
    double n[3];              /* unit normal pointing INTO the domain */
    double vel;               /* kinematic velocity along n (drive_wall) */
    double mu_t, mu_r;        /* frictionless by default */
    int32_t id, pad;          /* wall id in contact keys: 2*axis + side (0:-x 1:+x ... 5:+z) */
} or_wall;

#define OR_MAX_BOX 8
/* Rigid plate = union of axis-aligned boxes, translated only (reading R18). */
typedef struct {
    int32_t nbox, pad;
    double lo[OR_MAX_BOX][3], hi[OR_MAX_BOX][3];   /* box corners relative to pos */
    double pos[3], vel[3];
    double mass, mu_t, mu_r;
    int32_t mode[3];          /* per axis: 0 locked, 1 velocity-driven, 2 force-driven */
    int32_t pad2;
    double target[3];         /* m/s (velocity axis) or N (force axis) */
    double ramp[3];           /* linear ramp time of a velocity target */
    double t0[3];             /* time the drive started */
    double force[3];          /* out: contact reaction on the plate of the last step [N] */
    int32_t limit[3];         /* velocity axis with motor force limits (Eq. 4) */
    int32_t pad3;
    double fmin[3], fmax[3];  /* lambda_min, lambda_max [N] (used when limit[k]) */
    double motor[3];          /* out: the axis force of the last step [N] (target of a force axis) */
} or_plate;

/* A contact (output) or a history record (input; only key and P are read).
 * key = (key_a << 32) | key_b; key_a = smaller particle gid; key_b = partner gid, or
 * 2^32-16+w for box wall w, or 2^32-4096+16p+b for box b of plate p.
 * n points from body a (particle, smaller gid) to body b. P = (P_n, P_t[3], P_r[3]) [N s]. */
typedef struct {
    uint64_t key;
    double n[3];
    double delta;
    double P[7];
} or_contact;

typedef struct {
    int64_t n;                /* particles */
    double *x, *v, *w;        /* 3n each (in/out): position, velocity, angular velocity */
    const double *r;          /* n radii */
    const uint32_t *gid;      /* n unique ids (< 2^32-4096) */
    int32_t n_walls, n_plates;
    or_wall *walls;
    or_plate *plates;
    double time;
} or_world;

typedef struct {
    int64_t n_contacts, n_pp, n_wall, n_plate, n_degenerate;
    int32_t impact_fired, pad;
    double ke;                /* kinetic energy after the step */
    double max_v;             /* max |v| after the step */
    double max_normal_residual;   /* max |min(P_n, u_n + S P_n - b)| at the end of the solve */
    double max_cone_excess;   /* max(|P_t| - mu_t P_n, |P_r| - mu_r R* P_n) */
} or_report;

/* sphere mass and inertia from diameter: m = rho*pi*d^3/6, I = m d^2/10 */
void or_mass_inertia(double d, double rho, double *m, double *I);
/* effective contact parameters. db <= 0 means a flat tool (d* = da). */
void or_contact_params(double da, double db, double Ea, double Eb, double nua, double nub,
                       double e_H, double *Estar, double *dstar, double *kn, double *eps_n);
/* refinement planner (Eq. 1 and layers; Eqs. 8-10) */
double or_profile_diameter(double d_min, double d_max, double gamma, double depth);
int32_t or_layer_schedule(double d_min, double d_max, double r, double eta,
                          double *d_out, double *z_out, int32_t cap);
double or_contact_network_length(double d_min, double d_max, double r, double eta, double h);
int32_t or_solver_iterations(double n_d, double eps);
double or_planned_timestep(double d, double eps, double rho, double sigma);

/* SURVEY §8(c) binning mode: particle pairs from a uniform cell list instead of all N^2 pairs
 * (identical contact set and order; off by default) */
void or_set_binning(int32_t on);

/* brute-force O(N^2) detection: contacts sorted by key; returns 0 or -1 (cap) */
int32_t or_detect(const or_world *w, const or_params *p, or_contact *out, int64_t cap,
                  int64_t *n_out, int64_t *n_degenerate);

/* brute-force contacts of the particles idx[0..nidx) only (walls too; plates not included),
 * deduplicated and sorted by key: sampled pair-set checks on full-size beds */
int32_t or_contacts_of(const or_world *w, const int64_t *idx, int64_t nidx, or_contact *out, int64_t cap,
                       int64_t *n_out);

/* Colouring of the contact graph for the Gauss-Seidel ordering: contacts that
 * share a particle conflict.  Priority pi(c) = splitmix64(key(c)) (ties: smaller key first);
 * contacts are coloured greedily in decreasing priority, each with the smallest colour not used
 * by an already-coloured conflicting contact.  a[c], b[c]: particle indices (b < 0: wall or
 * plate).  color[c] out; returns the number of colours, or -1 if more than 256 are needed. */
int32_t or_color_contacts(int64_t nc, const uint64_t *key, const int64_t *a, const int64_t *b, int64_t n_particles,
                          int32_t *color);
uint64_t or_splitmix64(uint64_t x);

/* one full time step: detection, impact stage, SPOOK rows, warm start,
 * n_it Jacobi sweeps, integration, plates/walls.  hist (any order) supplies the warm start.
 * out receives the step's contacts with final impulses, sorted by key (= next history).
 * F, T (3n, may be NULL) receive per-particle contact force and torque (P/h sums).
 * Returns 0, -1 (out cap too small) or -2 (NaN/Inf). */
int32_t or_step(or_world *w, const or_params *p, const or_contact *hist, int64_t n_hist,
                or_contact *out, int64_t cap, int64_t *n_out, double *F, double *T,
                or_report *rep);

#ifdef __cplusplus
}
#endif
#endif
