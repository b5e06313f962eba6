// common.cuh -- device data layout and helpers shared by the CUDA kernels of libdem.so.
//
// Layout in HBM, all particle arrays in the rebuild's sorted (level, Morton)
// order:
//   pos   double4[N]  (x, y, z, r)
//   vel   double4[N]  (vx, vy, vz, c/m)      ping-pong x2, c = contact count (mass splitting)
//   ang   double4[N]  (wx, wy, wz, c/I)      ping-pong x2
//   gid   uint32[N]
// Contacts (compacted every step, in candidate order = sorted by (i, j)):
//   cij   uint2  (i, j)   j = particle, or PARTNER_EXT|code for walls/plate boxes
//   geo   G4 (n.xyz, mu_r R*)   n from i to j                     (G4 = float4 | double4)
//   row   R4 (Sigma-hat, b, la, lb)   la = r_i - delta/2, lb = r_j - delta/2   (R4 likewise)
//   cdel  double delta (rows and getters only)
//   Pa/Pb P4 (P_n, P_t.xyz) / (P_r.xyz, 0)   ping-pong x2          (P4 = float4 | double4)
// Incidence (half-contact CSR, per particle): inc uint2 (contact | B_SIDE, partner).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DEM_MAX_LEVELS 8
#define DEM_MAX_PLATES 8
#define DEM_MAX_BOXES 8
#define PARTNER_EXT 0x80000000u          // partner is not a particle
#define PARTNER_PLATE 0x00000100u        // ext code: plate box = EXT|PLATE|(p<<4)|b ; wall = EXT|w
#define B_SIDE 0x80000000u               // incidence entry: this particle is body b of the contact
#define INC_CMASK 0x7FFFFFFFu            // incidence entry: contact index bits
#define CCAND_FLIP 0x80000000u           // ccand entry: the contact's (a, b) is its candidate (j, i)

// Canonical orientation of a particle pair: body a = the smaller gid, so every
// decomposition evaluates a contact with the same operands in the same order.
__device__ __forceinline__ bool cand_flip(uint2 ij, const uint32_t *__restrict__ gid)
{
    return !(ij.y & PARTNER_EXT) && gid[ij.y] < gid[ij.x];
}
// sort key of an incidence partner: its gid; boundary bodies after all particles, by code
__device__ __forceinline__ uint64_t partner_key(uint32_t p, const uint32_t *__restrict__ gid)
{
    return (p & PARTNER_EXT) ? (1ull << 32) + (p & ~PARTNER_EXT) : (uint64_t)gid[p];
}
#define WALL_KEY_BASE 0xFFFFFFF0u        // public key of wall w: 2^32-16+w
#define PLATE_KEY_BASE 0xFFFFF000u       // public key of plate p box b: 2^32-4096+16p+b
#define FIXED_SCALE 1099511627776.0      // 2^40: int64 fixed point for plate impulse sums
#define NB_SLOTS (DEM_MAX_PLATES + 6)    // boundary-body sums: plates 0..7, walls 8..13
#define HUB_SCALE 4503599627370496.0     // 2^52: int64 fixed point of the per-sweep plate increments

// Storage precision of the contact arrays: -DDEM_P64 / -DDEM_G64 / -DDEM_R64
// store impulses / normals / row constants as fp64 instead of fp32 (all row arithmetic is fp64).
// The shipped build uses G64 + R64 (fp32 impulses), chosen by measured parity.
#ifdef DEM_P64
#error "DEM_P64 was retired: contact-array impulses are float4 (the sweep's item records choose their own precision)"
#endif
typedef float4 P4;
#ifdef DEM_G64
typedef double4 G4;
#else
typedef float4 G4;
#endif
#ifdef DEM_R64
typedef double4 R4;
#else
typedef float4 R4;
#endif
__host__ __device__ __forceinline__ P4 mkP4(double a, double b, double c, double d)
{
#ifdef DEM_P64
    return make_double4(a, b, c, d);
#else
    return make_float4((float)a, (float)b, (float)c, (float)d);
#endif
}
__host__ __device__ __forceinline__ G4 mkG4(double a, double b, double c, double d)
{
#ifdef DEM_G64
    return make_double4(a, b, c, d);
#else
    return make_float4((float)a, (float)b, (float)c, (float)d);
#endif
}
__host__ __device__ __forceinline__ R4 mkR4(double a, double b, double c, double d)
{
#ifdef DEM_R64
    return make_double4(a, b, c, d);
#else
    return make_float4((float)a, (float)b, (float)c, (float)d);
#endif
}
// value as stored in a P4 slot
__host__ __device__ __forceinline__ double rndP(double x)
{
#ifdef DEM_P64
    return x;
#else
    return (double)(float)x;
#endif
}

// Impulse storage: p_ld converts a stored value to double (exact), p_rnd rounds a double to the
// storage precision, writes it to the slot and returns it as a double (the value the velocity
// update must use so that momentum stays consistent with the stored impulses).  (An integer
// bit-manipulation version that keeps the F2F conversions off the XU pipe was measured: the XU
// pipe was not the limiter and it cost 36 % more instructions.)
#ifdef DEM_P64
__device__ __forceinline__ double p_ld(double v) { return v; }
__device__ __forceinline__ double p_rnd(double x, double &st)
{
    st = x;
    return x;
}
#else
__device__ __forceinline__ double p_ld(float f) { return (double)f; }
__device__ __forceinline__ double p_rnd(double x, float &st)
{
    st = (float)x;
    return (double)st;
}
#endif

// 256-bit global accesses (LDG.E.256 / STG.E.256 on sm_100a): one instruction and one sector
// per lane for a 32-byte record, instead of two 128-bit accesses that each touch the sector.
// ld4g is the non-coherent path: only for data the kernel does not write.
__device__ __forceinline__ double4 ld4g(const double4 *p)
{
    double4 v;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld4g(const float4 *p) { return __ldg(p); }
__device__ __forceinline__ void st4g(double4 *p, const double4 v)
{
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                 : "memory");
}

struct GridLevel {
    double ox, oy, oz;     // origin
    double cell;           // cell edge = 2 r_max(L) + skin
    double rmax;           // largest radius in the level
    int nx, ny, nz;        // cells per axis
    int present;           // level has particles
    uint64_t offset;       // first slot of the level in the dense cell tables
};

struct GridParams {
    int nlev;
    int bits;              // Morton bits per axis
    double rmin;           // level thresholds: L = #{k >= 1 : r >= rmin 2^k}
    double skin;
    GridLevel lv[DEM_MAX_LEVELS];
};

// Boundary bodies: box walls (kinematic along their normals) and translating plates.
struct DevBoundary {
    double wp[6][3];       // wall point
    double wn[6][3];       // inward normal
    double wvel[6];        // velocity along the inward normal
    int wpresent[6];
    double wall_mu_t, wall_mu_r;
    int n_plates;
    int mono;                           // monolithic force-driven plate axes (solver.plate_coupling)
    int nbox[DEM_MAX_PLATES];
    double lo[DEM_MAX_PLATES][DEM_MAX_BOXES][3], hi[DEM_MAX_PLATES][DEM_MAX_BOXES][3];
    double ppos[DEM_MAX_PLATES][3], pvel[DEM_MAX_PLATES][3];
    double pmass[DEM_MAX_PLATES], pmu_t[DEM_MAX_PLATES], pmu_r[DEM_MAX_PLATES];
    int mode[DEM_MAX_PLATES][3];
    double target[DEM_MAX_PLATES][3], ramp[DEM_MAX_PLATES][3], t0[DEM_MAX_PLATES][3];
    double pforce[DEM_MAX_PLATES][3];   // reaction of the last step [N]
    // motor force limits of velocity axes (Eq. 4: lambda_min <= lambda_j <= lambda_max)
    int plimit[DEM_MAX_PLATES][3];
    double pfmin[DEM_MAX_PLATES][3], pfmax[DEM_MAX_PLATES][3];
    double pmotor[DEM_MAX_PLATES][3];   // motor / constraint force of the last step [N]
    double wforce[6][3];                // wall reactions of the last step [N]
    int64_t wcount[6];
    int64_t pcount[DEM_MAX_PLATES];
    double time;
    // references at the last rebuild (trigger)
    double wp_ref[6][3], ppos_ref[DEM_MAX_PLATES][3];
};

struct SolveParams {
    double h, Ups, e_H, k_lin, Es, rho;
    double mu_t, mu_r, e_rest, v_imp;
    double g[3];
    int rolling_dims;
    int hertz;             // 1: e_H = 5/4 (sqrt(delta)); 0: linear
    double Cs;             // Sigma-hat constant: hertz 12 Ups/(h^2 e_H E*), linear 4 Ups/(h^2 e_H k_lin)
};

// SPOOK regularisation of the Hertz-mapped normal row in impulse units (reading R4):
// Sigma-hat = 4 Ups/(h^2 e_H k_n delta^(2 e_H - 2)), k_n = E* sqrt(d*)/3, d* = 2 R*
//           = Cs / sqrt(2 R* delta)                       (e_H = 5/4)
// linear model (reading R3): Sigma-hat = 4 Ups/(h^2 e_H k_lin) = Cs
#define spook_sigma(sp, Rs, delta) ((sp).hertz ? (sp).Cs * rsqrt64(2.0 * (Rs) * (delta)) : (sp).Cs)

// per-step scalars read back by the host once or twice per step
struct StepScalars {
    unsigned int n_contacts;
    unsigned int impact;          // any contact with u_n^- < -v_imp
    unsigned int n_degenerate;
    unsigned int n_pp, n_wall, n_plate;
    unsigned int nan_flag;
    unsigned int pad;
    unsigned long long max_disp_bits;   // max |x - x_ref| (double bits; non-negative -> ordered)
    unsigned long long max_v_bits;
    unsigned long long max_res_bits;    // max normal complementarity residual (report)
    unsigned long long max_cone_bits;   // max cone excess (report)
    double ke;
    double bnd_disp;
};

// ------------------------------------------------------------------ small double3 helpers
struct d3 { double x, y, z; };
__device__ __forceinline__ d3 mk(double x, double y, double z) { return d3{x, y, z}; }
__device__ __forceinline__ d3 operator+(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ d3 operator-(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ d3 operator*(double s, d3 a) { return d3{s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ d3 cross(d3 a, d3 b)
{
    return d3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// fp64 reciprocal: MUFU.RCP64H estimate + two Newton steps (relative error ~1e-16; operands
// are positive and finite: split weights, regularised diagonals)
__device__ __forceinline__ double rcp64(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}


// 1/sqrt(x) for x > 0: MUFU.RSQ64H estimate + two fp64 Newton steps (relative error ~1e-16)
__device__ __forceinline__ double rsqrt64(double x)
{
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = r * (1.5 - 0.5 * x * r * r);
    return r * (1.5 - 0.5 * x * r * r);
}

// 1/sqrt(x) for x > 0 with ONE Newton step (relative error ~1e-14): where the result only scales
// an iterate (cone projections, the SPOOK regularisation of a sweep), not a geometric quantity
__device__ __forceinline__ double rsqrt64_1(double x)
{
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r * (1.5 - 0.5 * x * r * r);
}

// R* = r_a r_b / (r_a + r_b) (d* = 2 R*): one definition for every kernel
__device__ __forceinline__ double rstar(double ra, double rb) { return ra * rb * rcp64(ra + rb); }

// Geometry of an active particle pair (d2 > 0 already established by the exact predicate):
// n = (x_b - x_a)/d, delta = r_a + r_b - d.  One instruction sequence used by the narrow phase
// and re-evaluated by the sweeps from the same positions, so both give bit-identical n, delta.
__device__ __forceinline__ void pair_geom(const double4 A, const double4 B, d3 &n, double &delta)
{
    const double dx = __dsub_rn(B.x, A.x), dy = __dsub_rn(B.y, A.y), dz = __dsub_rn(B.z, A.z);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    const double id = rsqrt64(d2);
    n = d3{dx * id, dy * id, dz * id};
    delta = __dsub_rn(__dadd_rn(A.w, B.w), __dmul_rn(d2, id));
}

// exact-sequence fp64 helpers (no FMA contraction) for predicates shared bit-for-bit with
// the fixed IEEE operation order of DESIGN.md reading R14
__device__ __forceinline__ double dist2_rn(double dx, double dy, double dz)
{
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Wall or plate-box contact of particle A (code = partner & ~PARTNER_EXT).  Walls: signed
// distance s = (X - p_w).n_w < r, n = -n_w, delta = r - s.  Plate boxes: closest point q of the
// box, n = (q - X)/|q - X|, delta = r - |q - X|; centre inside (reading R19): exit through the
// nearest face, delta = r + depth.  Returns 1 in contact, 0 not.  Also re-evaluated by the
// sweeps (boundary positions are fixed during a step's sweeps).
__device__ __forceinline__ int ext_geom(const double4 A, uint32_t code, const DevBoundary *bnd, d3 &n, double &delta)
{
    const double X[3] = {A.x, A.y, A.z};
    const double r = A.w;
    if (!(code & PARTNER_PLATE)) {
        const int w = (int)code;
        const double s = __dadd_rn(__dadd_rn(__dmul_rn(__dsub_rn(X[0], bnd->wp[w][0]), bnd->wn[w][0]),
                                             __dmul_rn(__dsub_rn(X[1], bnd->wp[w][1]), bnd->wn[w][1])),
                                   __dmul_rn(__dsub_rn(X[2], bnd->wp[w][2]), bnd->wn[w][2]));
        if (!(s < r)) return 0;
        n = d3{-bnd->wn[w][0], -bnd->wn[w][1], -bnd->wn[w][2]};
        delta = __dsub_rn(r, s);
        return 1;
    }
    const int p = (code >> 4) & 0xF, b = code & 0xF;
    double lo[3], hi[3], dq[3];
    for (int k = 0; k < 3; k++) {
        lo[k] = __dadd_rn(bnd->ppos[p][k], bnd->lo[p][b][k]);
        hi[k] = __dadd_rn(bnd->ppos[p][k], bnd->hi[p][b][k]);
        const double q = X[k] < lo[k] ? lo[k] : (X[k] > hi[k] ? hi[k] : X[k]);
        dq[k] = __dsub_rn(q, X[k]);
    }
    const double d2 = dist2_rn(dq[0], dq[1], dq[2]);
    if (d2 > 0.0) {
        if (!(d2 < __dmul_rn(r, r))) return 0;
        const double d = __dsqrt_rn(d2);
        n = d3{__ddiv_rn(dq[0], d), __ddiv_rn(dq[1], d), __ddiv_rn(dq[2], d)};
        delta = __dsub_rn(r, d);
        return 1;
    }
    double best = INFINITY, sg = 1.0;
    int bk = 0;
    for (int k = 0; k < 3; k++) {
        const double dl = __dsub_rn(X[k], lo[k]), dh = __dsub_rn(hi[k], X[k]);
        if (dl < best) { best = dl; bk = k; sg = 1.0; }
        if (dh < best) { best = dh; bk = k; sg = -1.0; }
    }
    n = d3{bk == 0 ? sg : 0.0, bk == 1 ? sg : 0.0, bk == 2 ? sg : 0.0};
    delta = __dadd_rn(r, best);
    return 1;
}


__host__ __device__ __forceinline__ int level_of(double r, double rmin, int nlev)
{
    int L = 0;
    double t = rmin;
    for (int k = 1; k < nlev; k++) {
        t = t * 2.0;
        if (r >= t) L = k;
    }
    return L;
}

__device__ __forceinline__ uint64_t spread3(uint32_t v)
{
    uint64_t x = v & 0x1fffff;   // 21 bits
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}
__device__ __forceinline__ uint32_t compact3(uint64_t x)
{
    x &= 0x1249249249249249ULL;
    x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ULL;
    x = (x ^ (x >> 4)) & 0x100f00f00f00f00fULL;
    x = (x ^ (x >> 8)) & 0x1f0000ff0000ffULL;
    x = (x ^ (x >> 16)) & 0x1f00000000ffffULL;
    x = (x ^ (x >> 32)) & 0x1fffffULL;
    return (uint32_t)x;
}

__device__ __forceinline__ int cell_coord(double x, double o, double c, int n)
{
    double f = floor((x - o) / c);
    int i = (f < 0.0) ? 0 : (f > (double)(n - 1) ? n - 1 : (int)f);
    return i;
}

// ------------------------------------------------------------------ host-side launchers
struct LaunchCounter { long long *count; };

// scan.cu
size_t scan_temp_bytes(int64_t n);
// exclusive scan of n uint32 (in-place allowed); out[n] = total.  temp from scan_temp_bytes.
void scan_u32(const uint32_t *in, uint32_t *out, int64_t n, void *temp, cudaStream_t s, long long *launches);

// radix_sort.cu: stable LSD sort of (key, val) pairs on bits [0, nbits); result in keys[0], vals[0]
size_t sort_temp_bytes(int64_t n);
void radix_sort_u64(uint64_t *keys[2], uint32_t *vals[2], int64_t n, int nbits, void *temp,
                    cudaStream_t s, long long *launches);
