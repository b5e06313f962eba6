/*
 * dem.h -- C-ABI of the B200-native nonsmooth-DEM time step (libdem.so).
 *
 * The library implements one time step of the discrete element method of
 * Pogulis & Servin, "Local particle refinement in terramechanical simulations"
 * (arXiv 2501.05300; /root/reference/PAPER.md, cited "P:line"): a bed of spheres whose size
 * grows with depth (Eq. 1), stepped by the time-implicit (nonsmooth) DEM of
 * contact detection every step, Hertz-mapped SPOOK normal rows
 * (P:127-129), Coulomb and rolling-resistance cones, a Newton
 * impact stage, and a warm-started projected iterative solve run here as a
 * deterministic Jacobi sweep on the GPU.  Readings of silent/garbled passages: DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - SI units, z up, gravity is a solver parameter (default (0,0,-9.81)); "depth" = z_top - z.
 *  - All state is double precision (fp64 x, v, w); contact normals and row constants are
 *    stored in fp64, impulses in fp32, and all contact-row arithmetic is fp64.
 *  - Particles are identified by a caller-chosen unique gid (uint32 < 2^32-4096).  Every
 *    getter returns particles in ascending gid order and contacts in ascending key order.
 *  - A contact key is (key_a << 32) | key_b with key_a = the smaller gid of the pair and
 *    key_b = the other gid, or 2^32-16+w for box wall w, or 2^32-4096+16p+b for box b of
 *    plate p.  The normal points from body a to body b; P = (P_n, P_t[3], P_r[3]) in N s is
 *    the impulse body b receives (body a receives the opposite).
 *  - Ownership: the context owns all device memory (allocated through dem_dist_desc.alloc
 *    when given, else cudaMalloc).  No caller pointer is retained after a call returns.
 *    Buffers passed to getters/setters are host memory unless the view's on_device is 1.
 *  - Errors: every call returns a dem_status; DEM_ERR_INVALID leaves the context unchanged;
 *    dem_last_error() returns a human-readable reason.  A step that produces NaN/Inf returns
 *    DEM_ERR_DIVERGED and restores the state of the beginning of that step (S:385 atomicity).
 *  - Concurrency: one host thread per context; contexts on different devices are independent.
 *  - Determinism: for identical inputs the results are bit-identical run to run (no float
 *    atomics anywhere; all reductions are in a fixed order or in int64 fixed point).
 */
#ifndef DEM_H
#define DEM_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dem_ctx dem_ctx;

typedef enum {
    DEM_OK = 0,
    DEM_ERR_INVALID = 2,   /* bad argument or descriptor; nothing changed */
    DEM_ERR_DIVERGED = 3,  /* NaN/Inf in the step; state rolled back to the step start */
    DEM_ERR_STATE = 4,     /* call out of order (e.g. forces before any step) */
    DEM_ERR_CUDA = 5,      /* CUDA runtime error (message in dem_last_error) */
    DEM_ERR_NCCL = 6,      /* reserved: multi-GPU communicator error */
    DEM_ERR_OOM = 7        /* device allocation failed */
} dem_status;

/* Particle material (BASELINE configs: rho 2600, E 10 MPa, nu .3, mu .4/.1, e .5). */
typedef struct {
    double density, youngs, poisson;   /* E* = E/(2(1-nu^2)) for identical materials */
    double mu_t, mu_r;                 /* Coulomb |P_t| <= mu_t P_n; rolling |P_r| <= mu_r R* P_n */
    double restitution;                /* Newton impact law coefficient */
} dem_material;

/* Solver settings. */
typedef struct {
    double dt;                 /* time step h > 0 */
    int32_t n_iter;            /* Jacobi sweeps per step, >= 1 (Eq. 8 via dem_plan_iterations) */
    int32_t n_iter_impact;     /* impact-stage sweeps; <= 0 -> n_iter */
    double hertz_exp;          /* e_H: 1.25 (Hertz) or 1.0 (linear model) */
    double k_lin;              /* linear stiffness [N/m], required iff hertz_exp == 1 */
    double damping_steps;      /* SPOOK damping time tau = damping_steps * dt (4.5) */
    double v_impact;           /* impact threshold [m/s]; < 0 -> 20 |g| dt; >= 1e30 off */
    double gravity[3];
    int32_t rolling_dims;      /* 3: rolling row on the full relative spin (default); 2: tangential */
    int32_t ordering;          /* 0: Jacobi sweep with mass splitting (default, reading R2);
                                  1: coloured projected Gauss-Seidel (P:134 PGS):
                                  contacts coloured greedily in SplitMix64(key) priority, swept colour
                                  by colour with the real masses (single undecomposed context only) */
    double skin;               /* Verlet skin [m] of the candidate list; <= 0 -> 0.1 r_min */
    int32_t reduction;         /* kept for the ABI; 0 and 1 are identical.  The Jacobi sweep sums each
                                  particle's contact increments exactly (int64 fixed point at a scale
                                  chosen from the particle's own weights, sweep.cu), so trajectories
                                  are bit-identical for any number of GPUs/slabs and
                                  run to run; values other than 0/1 -> DEM_ERR_INVALID */
    int32_t plate_coupling;    /* force-driven plate axes: 0 staggered after the solve (reading R18,
                                  default); 1 monolithic -- the axis is a body of the impact and
                                  main-stage solves (reading R18b): V += (h F + sum of
                                  its contacts' warm-start impulses)/M before the sweeps, V += sum of
                                  the sweep's impulse increments / M after each, x += h V at the end
                                  (Jacobi ordering only) */
} dem_solver;

/* Container: axis-aligned box; wall w = 2*axis + side (0:-x 1:+x 2:-y 3:+y 4:-z 5:+z). */
typedef struct {
    double lo[3], hi[3];
    uint32_t wall_mask;        /* bit w set -> wall w present */
    uint32_t pad0;
    double wall_mu_t, wall_mu_r;   /* walls are frictionless in the paper */
} dem_box;

/* Particle arrays, caller order (host unless on_device). */
typedef struct {
    int64_t n;
    const double *pos;         /* 3n */
    const double *radius;      /* n, > 0 */
    const double *vel;         /* 3n or NULL (zero) */
    const double *angvel;      /* 3n or NULL (zero) */
    const uint32_t *gid;       /* n unique, < 2^32-4096, or NULL (0..n-1) */
    int32_t on_device;
    int32_t pad0;
} dem_particles;

/* On-device bed generator (refinement profiles P:65-78, Eq. 1 and Fig. 2; size
 * jitter P:161).  The bed fills the box from the bottom face up to the top face; depth is
 * measured down from box.hi[2].
 *   kind 0 bands: band k spans depths [band_bottom_depth[k-1], band_bottom_depth[k]) (band 0
 *          from depth 0) with nominal radius band_r_nom[k]; an FCC lattice per band with
 *          nearest-neighbour distance spacing_factor * r_nom, kept 1.1 r_nom from the band faces
 *          and the walls.
 *   kind 1 linear profile (Eq. 1): d(depth) = d_min + gamma depth, capped at d_max; square
 *          lattice planes from the bottom up, in-plane spacing spacing_factor * r(z), vertical gap
 *          spacing_factor (r_k + r_k+1) / 2.
 *   kind 2 layer schedule (Fig. 2): layers n = 0, 1, ... from the top with d_n = d_min ratio_r^n
 *          and thickness eta d_n while d_n < d_max, d_max below; generated as kind 0 bands.
 * Jitter: each coordinate += pos_jitter r_nom U(-1, 1), radius = r_nom U(1 - size_jitter,
 * 1 + size_jitter), from Philox4x32-10 keyed by seed with counter gid.  gids run plane by plane
 * from the bottom (then lattice sub-grid, y, x).  With world_size > 1 every rank generates the
 * sites of its slab (by lattice x; the outer slabs are open) under their global gids, so the
 * union over ranks is the single-rank bed.  Velocities start at zero. */
typedef struct {
    int32_t kind;                      /* 0 bands, 1 linear profile, 2 layer schedule */
    int32_t n_bands;                   /* kind 0: number of bands (<= 64) */
    const double *band_bottom_depth;   /* kind 0: n_bands increasing depths [m] (host memory) */
    const double *band_r_nom;          /* kind 0: n_bands nominal radii [m] (host memory) */
    double d_min, gamma, d_max;        /* kinds 1, 2: diameters [m], gamma = dd/ddepth */
    double ratio_r, eta;               /* kind 2: size ratio between layers > 1, layer thickness / d */
    double spacing_factor;             /* lattice distance / r_nom; 2.25 leaves every pair apart */
    double pos_jitter, size_jitter;    /* 0.01 and 0.10 */
    uint64_t seed;
} dem_generator;

typedef struct {
    size_t struct_size;        /* sizeof(dem_bed_desc): ABI version check */
    dem_material mat;
    dem_solver solver;
    dem_box box;
    dem_particles parts;       /* source 0 */
    int32_t source;            /* 0: the particle arrays, 1: the generator */
    int32_t pad0;
    dem_generator gen;         /* source 1 */
} dem_bed_desc;

/* Process / device plumbing (PyTorch provides memory, stream and process group) and the x-slab
 * domain decomposition.  world_size > 1: each rank owns the
 * particles of its slab [slab_lo, slab_hi) along x (ranks ordered by x, neighbours rank +- 1)
 * and passes only those to dem_create_bed; the library keeps ghost copies of the neighbours'
 * particles within 2 r_max + 2 skin of the shared faces, refreshes their velocities after every
 * Jacobi sweep, and moves ownership at each rebuild.  create, step and destroy are then
 * collective over the ranks.  The outer faces of rank 0 and rank world_size-1 are open (they own
 * whatever lies beyond the box).  world_size 1 with a transport (nccl_unique_id or loopback set)
 * runs the decomposed code path on one rank with no neighbours (transport self-test). */
typedef struct {
    int32_t rank, world_size;
    const void *nccl_unique_id;        /* transport 0, world_size > 1: the 128-byte ncclUniqueId of
                                          rank 0 (dem_nccl_unique_id), broadcast by the caller */
    void *cuda_stream;                 /* cudaStream_t all work is issued on; NULL -> own stream */
    void *(*alloc)(size_t bytes, void *alloc_ctx);   /* NULL -> cudaMalloc */
    void (*free)(void *ptr, void *alloc_ctx);
    void *alloc_ctx;
    double slab_lo, slab_hi;           /* world_size > 1: this rank's slab along x, slab_lo < slab_hi */
    int32_t transport;                 /* 0: NCCL, one process per GPU; 1: in-process loopback group */
    int32_t pad0;
    void *loopback;                    /* transport 1: dem_loopback_create handle shared by the ranks,
                                          each rank driven by its own host thread */
} dem_dist_desc;

typedef struct {
    int64_t step;              /* steps taken since create */
    double time;
    int64_t n_contacts, n_pp, n_wall, n_plate, n_degenerate, n_candidates;
    int32_t impact_fired;      /* 1 if the Newton impact stage ran in this step */
    int32_t rebuilt;           /* 1 if the sort/grid/candidate list was rebuilt before this step */
    double ke;                 /* kinetic energy after the step [J] */
    double max_v;              /* max |v| after the step */
    double max_disp;           /* max displacement since the last rebuild [m] */
    int32_t n_iter, n_iter_impact;
    int32_t n_colors;          /* Gauss-Seidel ordering: colours of the step's contact graph (else 0) */
    int32_t pad0;
    double max_normal_residual; /* max over contacts of |min(P_n, u_n + Sigma P_n - b)| at the final
                                   velocities [N s or m/s mix, as the row] (S:365 convergence report) */
    double max_cone_excess;    /* max(0, |P_t| - mu_t P_n, |P_r| - mu_r R* P_n) [N s] */
} dem_step_report;

/* State exchange, ascending gid order; n = capacity in, count out. */
typedef struct {
    int64_t n;
    double *pos;               /* 3n */
    double *vel;               /* 3n */
    double *angvel;            /* 3n */
    double *radius;            /* n */
    uint32_t *gid;             /* n */
    int32_t on_device;
    int32_t pad0;
} dem_state_view;

typedef struct {
    int64_t n;                 /* capacity in, count out */
    uint64_t *key;             /* n, ascending */
    double *normal;            /* 3n (may be NULL for input) */
    double *delta;             /* n  (may be NULL for input) */
    double *P;                 /* 7n: P_n, P_t[3], P_r[3] */
    int32_t on_device;
    int32_t pad0;
} dem_contact_view;

typedef enum { DEM_AXIS_LOCKED = 0, DEM_AXIS_VELOCITY = 1, DEM_AXIS_FORCE = 2 } dem_axis_mode;

/* Rigid plate = union of <= 8 axis-aligned boxes (base + grousers), translation only. */
typedef struct {
    int32_t n_boxes, pad0;
    const double *lo, *hi;     /* 3*n_boxes corners relative to the plate position */
    double mass;               /* used by force-driven axes */
    double mu_t, mu_r;         /* plate-particle coefficients (same as inter-particle) */
} dem_plate_desc;

typedef struct {
    double pos[3], vel[3];
    double force[3];           /* contact reaction on the plate during the last step [N] */
    double motor_force[3];     /* axis force of the last step [N]: the target of a force axis; for
                                  velocity / locked axes the constraint (motor) force lambda_j that
                                  the drive applied (the required pull force) */
    int64_t n_contacts;
} dem_plate_state;

typedef struct {
    double ms_total;           /* device time of the timed phases since reset [ms] */
    double ms_detect;          /* narrow phase + compaction + incidence + rows */
    double ms_rebuild;         /* keys, sort, grid, broad phase, history carry */
    double ms_sweeps;          /* all Jacobi sweeps (main + impact) */
    double ms_integrate;
    int64_t n_sweep_launches;
    int64_t n_kernel_launches; /* every kernel this library launched */
    int64_t contact_sweeps;    /* sum over sweeps of the contact count */
    int64_t particle_sweeps;   /* sum over sweeps of the particle count */
} dem_timing;

/* Create a bed from particle arrays (P:155-161 beds are produced by synth/ generators).
 * Validates (DEM_ERR_INVALID): struct_size, material > 0, 0 <= nu < .5, dt > 0, n_iter >= 1,
 * radius > 0, unique gids, box lo < hi, decomposition fields (world_size > 1: particles inside the
 * slab; DEM_ERR_NCCL if the transport cannot be set up).  Builds the first candidate list. */
dem_status dem_create_bed(const dem_bed_desc *desc, const dem_dist_desc *dist, dem_ctx **out);

/* Advance n_steps >= 1 time steps.  `last` (may be NULL) gets the report of the
 * final step.  Synchronises the host once per step (impact/rebuild decisions). */
dem_status dem_step(dem_ctx *ctx, int32_t n_steps, dem_step_report *last);

/* Replace the solver settings (same validation as create), e.g. a coarse dt and few sweeps
 * for relaxing a generated bed before the production settings.  Takes effect at the
 * next step; the Verlet skin is kept. */
dem_status dem_set_solver(dem_ctx *ctx, const dem_solver *solver);

/* Copy particle state out (gid order).  view->n must be >= the owned particle count (else
 * DEM_ERR_INVALID with view->n set to it); on return view->n = the count.  Any field pointer may
 * be NULL: that field is not copied (the field mask of SURVEY §8(b)).  on_device selects device or
 * host buffers.  Decomposed: this rank's owned particles. */
dem_status dem_get_state(dem_ctx *ctx, dem_state_view *view);

/* Replace particle state (same gid set and radii as at create) and the contact history used
 * as warm start of the next step (hist may be NULL: no history).  Triggers a rebuild. */
dem_status dem_set_state(dem_ctx *ctx, const dem_state_view *state, const dem_contact_view *hist);

/* Contacts of the last step with final impulses, key order.  DEM_ERR_STATE before any step;
 * DEM_ERR_INVALID with view->n = required count if the capacity is too small. */
dem_status dem_get_contacts(dem_ctx *ctx, dem_contact_view *view);

/* Per-particle contact force F = sum(+-P_lin)/h and torque T (gid order, 3n each) of the last
 * step (O6).  on_device selects device or host buffers. */
dem_status dem_get_forces(dem_ctx *ctx, double *F, double *T, int32_t on_device);

/* Plates: add (all axes locked), drive one axis, read state.
 * dem_drive_plate: mode DEM_AXIS_VELOCITY is a motor G_j v = u_j(t) with u ramped linearly
 * from 0 to target over ramp_time from the call; its constraint force is limited to
 * [f_min, f_max] (Eq. 4; -INFINITY / INFINITY: unlimited).  Coupling is staggered (reading
 * R18): after each step the motor force lambda = m (u(t+h) - v)/h - F_contact is clamped to the
 * limits and the axis velocity for the next step is v + h (lambda + F_contact)/m (= u(t+h)
 * exactly when no limit is active).  At the call an unlimited velocity axis takes u at once (0 if
 * ramped), a limited one keeps its velocity.  Force axes (target in N) and locked axes ignore the
 * limits.
 * DEM_ERR_INVALID: bad plate/axis/mode, non-finite target, ramp_time < 0, NaN or f_min > f_max. */
dem_status dem_add_plate(dem_ctx *ctx, const dem_plate_desc *desc, const double pos[3], int32_t *plate_id);
dem_status dem_drive_plate(dem_ctx *ctx, int32_t plate, int32_t axis, int32_t mode,
                           double target /* m/s or N */, double ramp_time /* s, velocity mode */,
                           double f_min, double f_max /* N, velocity mode (Eq. 4) */);
dem_status dem_get_plate(dem_ctx *ctx, int32_t plate, dem_plate_state *out);

/* Change the particle set of a single context (the bed builder's emitter and trimming, SURVEY
 * NEXT-2).  dem_add_particles appends n particles (pos 3n, radius n, vel/angvel 3n or
 * NULL = 0, gid n: unique over the whole bed, < 2^32-4096; on_device: device pointers);
 * dem_remove_particles removes every particle whose coordinate `axis` lies outside [lo, hi] and
 * reports how many.  The state of the other particles and the contact history (the next step's
 * warm start) are kept; the next step rebuilds.  DEM_ERR_INVALID: bad arguments, a decomposed
 * context, or the validation of dem_create_bed (radius, finite positions, duplicate gid). */
dem_status dem_add_particles(dem_ctx *ctx, int64_t n, const double *pos, const double *radius, const double *vel,
                             const double *angvel, const uint32_t *gid, int32_t on_device);
dem_status dem_remove_particles(dem_ctx *ctx, int32_t axis, double lo, double hi, int64_t *n_removed);

/* Load balance of the x-slab decomposition; collective, a no-op without a
 * decomposition.  The owned particles' x are histogrammed over the box in n_bins >= 2 bins and
 * summed over the ranks; each interior face moves toward its particle-count quantile by at most
 * one Verlet skin (a particle that changes owner and all its last-step contacts, with their
 * impulse history, are then already held by its new owner: the trajectory stays bit-identical),
 * interior slabs stay at least one band wide.  Ownership moves at the next step's rebuild.
 * faces_out (may be NULL): the world_size - 1 new faces.  Call every M steps to converge. */
dem_status dem_rebalance(dem_ctx *ctx, int32_t n_bins, double *faces_out);

/* Kinematic box wall: velocity along its inward normal (shear-box / servo walls). */
dem_status dem_drive_wall(dem_ctx *ctx, int32_t wall, double normal_velocity);

/* Box wall state (walls: P:252; servo-controlled triaxial walls: P:166-202).
 * Wall w = 2 axis + side (0 -x, 1 +x, 2 -y, 3 +y, 4 -z, 5 +z); its plane passes through `point`
 * with inward unit `normal`.  force = contact reaction on the wall during the last step,
 * (1/h) sum over its contacts of (P_n n + P_t), an exact int64 sum over contacts and ranks (the
 * stress a wall carries is -force . normal / area).  DEM_ERR_INVALID: no such wall. */
typedef struct {
    double point[3], normal[3];
    double velocity;           /* along the inward normal [m/s] */
    double force[3];           /* [N] */
    int64_t n_contacts;
} dem_wall_state;
dem_status dem_get_wall(dem_ctx *ctx, int32_t wall, dem_wall_state *out);

/* Device-time accounting of the library's own kernels (CUDA events on the ctx stream). */
dem_status dem_set_timing(dem_ctx *ctx, int32_t enable);
dem_status dem_get_timing(dem_ctx *ctx, dem_timing *out);
dem_status dem_reset_timing(dem_ctx *ctx);

/* Diagnostic (not on the stepping path): time n >= 1 Jacobi sweeps of the shipped sweep kernel
 * (variant must be 0; sweep.cu) on the last step's contacts, from the current
 * velocities and the last step's final impulses with the main-stage rows.  Output: device ms per
 * sweep (CUDA events on the context's stream); *max_dv_rel is set to 0.  The particle state and
 * contact getters are unchanged.  DEM_ERR_STATE before any step; DEM_ERR_INVALID for n < 1, a
 * variant other than 0, a decomposed context or the Gauss-Seidel ordering. */
dem_status dem_bench_sweeps(dem_ctx *ctx, int32_t variant, int32_t n, double *ms_per_sweep, double *max_dv_rel);

/* Bytes one drive call (dem_drive_wall, dem_drive_plate) copies host -> device: the boundary
 * state is uploaded whole (accounting of end-to-end benchmarks).  Pure, never fails. */
int64_t dem_drive_upload_bytes(void);

/* Owned particles of this rank (all particles with world_size 1), and owned + ghost copies. */
int64_t dem_num_particles(const dem_ctx *ctx);
int64_t dem_num_local(const dem_ctx *ctx);

/* x-slab decomposition plumbing.  dem_nccl_unique_id writes a fresh 128-byte ncclUniqueId
 * (rank 0 calls it; DEM_ERR_NCCL if libnccl.so.2 cannot be loaded).  dem_loopback_create
 * returns a group through which world_size ranks of ONE process exchange ghosts with device
 * copies after host barriers (each rank's calls from its own thread); destroy it after every
 * rank's dem_destroy. */
dem_status dem_nccl_unique_id(void *out128);
void *dem_loopback_create(int32_t world_size);
void dem_loopback_destroy(void *group);

/* The cudaStream_t the context issues its work on. */
void *dem_stream(dem_ctx *ctx);

dem_status dem_destroy(dem_ctx *ctx);

/* Last error message of ctx (ctx == NULL: of the last failed create on this thread). */
const char *dem_last_error(const dem_ctx *ctx);

/* Host-only: number of particles the generator places in [slab_lo, slab_hi) of the lattice x
 * (pass -INFINITY, INFINITY for the whole bed).  DEM_ERR_INVALID for bad parameters. */
dem_status dem_generator_count(const dem_generator *gen, const dem_box *box, double slab_lo, double slab_hi,
                               int64_t *n);

/* ---- host-only planner helpers, pure functions ---- */
/* Eq. 1: d(z) = d_min + gamma z for z < z_max = (d_max - d_min)/gamma, else d_max. */
double dem_profile_diameter(double d_min, double d_max, double gamma, double depth);
/* Eq. 10: n_d = eta ln(d_max/d_min)/ln r + (h - z_max)/d_max, gamma = (r-1)/(r eta); h/d if uniform. */
double dem_contact_network_length(double d_min, double d_max, double r, double eta, double h);
/* Eq. 8: N_it = ceil(0.1 n_d / eps), at least 1. */
int32_t dem_plan_iterations(double n_d, double eps);
/* Eq. 9: dt = 0.5 sqrt(eps d / a), a = 3 sigma/(2 rho d). */
double dem_plan_timestep(double d, double eps, double rho, double sigma);

#ifdef __cplusplus
}
#endif
#endif
