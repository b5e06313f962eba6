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
#define WALL_KEY_BASE 0xFFFFFFF0u        // public key of wall w: 2^32-16+w
#define PLATE_KEY_BASE 0xFFFFF000u       // public key of plate p box b: 2^32-4096+16p+b
#define FIXED_SCALE 1099511627776.0      // 2^40: int64 fixed point for plate impulse sums

// Storage precision of the contact arrays: -DDEM_P64 / -DDEM_G64 / -DDEM_R64
// store impulses / normals / row constants as fp64 instead of fp32 (all row arithmetic is fp64).
// The shipped build uses G64 + R64 (fp32 impulses), chosen by measured parity.
#ifdef DEM_P64
typedef double4 P4;
#else
typedef float4 P4;
#endif
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
    int nbox[DEM_MAX_PLATES];
    double lo[DEM_MAX_PLATES][DEM_MAX_BOXES][3], hi[DEM_MAX_PLATES][DEM_MAX_BOXES][3];
    double ppos[DEM_MAX_PLATES][3], pvel[DEM_MAX_PLATES][3];
    double pmass[DEM_MAX_PLATES], pmu_t[DEM_MAX_PLATES], pmu_r[DEM_MAX_PLATES];
    int mode[DEM_MAX_PLATES][3];
    double target[DEM_MAX_PLATES][3], ramp[DEM_MAX_PLATES][3], t0[DEM_MAX_PLATES][3];
    double pforce[DEM_MAX_PLATES][3];   // reaction of the last step [N]
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
};

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

// exact-sequence fp64 helpers (no FMA contraction) for predicates shared bit-for-bit with
// the fixed IEEE operation order of DESIGN.md reading R14
__device__ __forceinline__ double dist2_rn(double dx, double dy, double dz)
{
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
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
