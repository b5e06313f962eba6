// generate.cu -- on-device bed generator (include/dem.h dem_generator): lattice beds
// whose particle size grows with depth (bands, the linear profile of Eq. 1, the layer
// schedule of Fig. 2) with the size jitter of P:161.
//
// The host lays out the lattice as a table of rectangular site grids (one per lattice plane and
// sub-grid), restricted to the rank's slab; one device thread per site then computes the site,
// its global gid, and the jitter from a Philox4x32-10 stream keyed by the seed with the gid as
// counter -- so a site gets the same particle whichever rank generates it.
#include <cmath>
#include <string>
#include <vector>

#include "../../include/dem.h"
#include "common.cuh"
#include "kernels.h"

struct GenPlane {
    double z, x0, y0, dx, dy, r;
    int32_t nx, ny, i0, ni;        // full grid nx x ny; this rank's columns [i0, i0 + ni)
    uint64_t gid0;                 // gid of site (0, 0)
    int64_t local0;                // first local index of this plane
};

static void fcc_band(double lo[3], double hi[3], double a, double r, std::vector<GenPlane> &P)
{
    const double A = a * std::sqrt(2.0);
    if (hi[2] < lo[2] || hi[0] < lo[0] || hi[1] < lo[1]) return;
    const int nz = (int)std::floor((hi[2] - lo[2]) / (0.5 * A) + 1e-9) + 1;
    for (int kz = 0; kz < nz; kz++) {
        const double z = lo[2] + 0.5 * A * kz;
        // FCC: half-planes alternate the sub-grids (0,0),(1/2,1/2) and (1/2,0),(0,1/2) in units of A
        const double off[2][2] = {{0.0, 0.0}, {0.5, 0.5}};
        const double offo[2][2] = {{0.5, 0.0}, {0.0, 0.5}};
        for (int b = 0; b < 2; b++) {
            const double bx = (kz % 2 ? offo[b][0] : off[b][0]) * A, by = (kz % 2 ? offo[b][1] : off[b][1]) * A;
            if (hi[0] - lo[0] - bx < -1e-12 || hi[1] - lo[1] - by < -1e-12) continue;
            GenPlane p{};
            p.z = z;
            p.x0 = lo[0] + bx;
            p.y0 = lo[1] + by;
            p.dx = p.dy = A;
            p.r = r;
            p.nx = (int)std::floor((hi[0] - p.x0) / A + 1e-9) + 1;
            p.ny = (int)std::floor((hi[1] - p.y0) / A + 1e-9) + 1;
            P.push_back(p);
        }
    }
}

// host: the lattice of the generator as grids, bottom up; gids and the slab restriction
static bool build_planes(const dem_generator &g, const dem_box &box, double slab_lo, double slab_hi,
                         std::vector<GenPlane> &P, int64_t &n_local, std::string &err)
{
    P.clear();
    const double H = box.hi[2] - box.lo[2];
    if (!(g.spacing_factor > 0) || g.pos_jitter < 0 || g.size_jitter < 0 || g.size_jitter >= 1 || !(H > 0)) {
        err = "generator: spacing_factor > 0, jitters >= 0, size_jitter < 1";
        return false;
    }
    std::vector<double> bot, rn;       // bands: bottom depth, nominal radius
    if (g.kind == 0) {
        if (g.n_bands < 1 || g.n_bands > 64 || !g.band_bottom_depth || !g.band_r_nom) { err = "generator: bands"; return false; }
        for (int k = 0; k < g.n_bands; k++) {
            if (!(g.band_r_nom[k] > 0) || (k && !(g.band_bottom_depth[k] > g.band_bottom_depth[k - 1])) ||
                !(g.band_bottom_depth[k] > 0)) { err = "generator: band depths increasing, radii > 0"; return false; }
            bot.push_back(g.band_bottom_depth[k]);
            rn.push_back(g.band_r_nom[k]);
        }
    } else if (g.kind == 2) {
        if (!(g.d_min > 0) || !(g.d_max >= g.d_min) || !(g.ratio_r > 1) || !(g.eta > 0)) { err = "generator: layer schedule"; return false; }
        double depth = 0.0, d = g.d_min;
        while (d < g.d_max && depth < H) {
            depth += g.eta * d;
            bot.push_back(std::min(depth, H));
            rn.push_back(0.5 * d);
            d *= g.ratio_r;
        }
        if (depth < H) { bot.push_back(H); rn.push_back(0.5 * g.d_max); }
    } else if (g.kind != 1) {
        err = "generator: kind 0, 1 or 2";
        return false;
    }
    if (g.kind != 1) {
        // bands bottom up
        for (int k = (int)bot.size() - 1; k >= 0; k--) {
            const double top = k ? bot[k - 1] : 0.0, r = rn[k], m = 1.1 * r;
            double lo[3] = {box.lo[0] + m, box.lo[1] + m, box.hi[2] - std::min(bot[k], H) + m};
            double hi[3] = {box.hi[0] - m, box.hi[1] - m, box.hi[2] - top - m};
            fcc_band(lo, hi, g.spacing_factor * r, r, P);
        }
    } else {
        if (!(g.d_min > 0) || !(g.d_max >= g.d_min) || g.gamma < 0) { err = "generator: linear profile"; return false; }
        auto rnom = [&](double z) {             // Eq. 1 with d = 2 r; depth from the top face
            const double depth = box.hi[2] - z;
            return 0.5 * std::min(g.d_min + g.gamma * std::max(depth, 0.0), g.d_max);
        };
        double z = box.lo[2] + 1.1 * rnom(box.lo[2]);
        for (int guard = 0; guard < 1000000; guard++) {
            const double rk = rnom(z);
            if (z + 1.1 * rk > box.hi[2]) break;
            const double m = 1.1 * rk, s = g.spacing_factor * rk;
            GenPlane p{};
            p.z = z;
            p.x0 = box.lo[0] + m;
            p.y0 = box.lo[1] + m;
            p.dx = p.dy = s;
            p.r = rk;
            p.nx = (int)std::floor((box.hi[0] - m - p.x0) / s + 1e-9) + 1;
            p.ny = (int)std::floor((box.hi[1] - m - p.y0) / s + 1e-9) + 1;
            if (p.nx > 0 && p.ny > 0) P.push_back(p);
            double zn = z + s;
            for (int it = 0; it < 4; it++) zn = z + 0.5 * g.spacing_factor * (rk + rnom(zn));
            z = zn;
        }
    }
    uint64_t gid = 0;
    n_local = 0;
    for (auto &p : P) {
        p.gid0 = gid;
        gid += (uint64_t)p.nx * (uint64_t)p.ny;
        // columns whose lattice x lies in [slab_lo, slab_hi)
        double a = std::ceil((slab_lo - p.x0) / p.dx), b = std::ceil((slab_hi - p.x0) / p.dx);
        a = std::isfinite(a) ? std::max(0.0, std::min(a, (double)p.nx)) : (slab_lo < 0 ? 0.0 : (double)p.nx);
        b = std::isfinite(b) ? std::max(0.0, std::min(b, (double)p.nx)) : (slab_hi > 0 ? (double)p.nx : 0.0);
        p.i0 = (int)a;
        p.ni = std::max(0, (int)b - (int)a);
        p.local0 = n_local;
        n_local += (int64_t)p.ni * p.ny;
    }
    if (gid >= (uint64_t)PLATE_KEY_BASE) { err = "generator: more sites than gids"; return false; }
    return true;
}

// ------------------------------------------------------------------ device
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k)
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += W0;
        k.y += W1;
    }
    return c;
}
__device__ __forceinline__ double u01(uint32_t x) { return ((double)x + 0.5) * 2.3283064365386963e-10; }

__global__ void k_generate(int64_t n, const GenPlane *__restrict__ P, int np, uint64_t seed, double pj, double sj,
                           double *__restrict__ x, double *__restrict__ r, uint32_t *__restrict__ gid)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    int lo = 0, hi = np - 1;                   // last plane with local0 <= q
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (P[mid].local0 <= q) lo = mid; else hi = mid - 1;
    }
    const GenPlane p = P[lo];
    const int64_t k = q - p.local0;
    const int j = (int)(k / p.ni), i = p.i0 + (int)(k % p.ni);
    const uint64_t g = p.gid0 + (uint64_t)j * (uint64_t)p.nx + (uint64_t)i;
    const uint4 u = philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0u, 0u),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    x[3 * q] = p.x0 + i * p.dx + pj * p.r * (2.0 * u01(u.x) - 1.0);
    x[3 * q + 1] = p.y0 + j * p.dy + pj * p.r * (2.0 * u01(u.y) - 1.0);
    x[3 * q + 2] = p.z + pj * p.r * (2.0 * u01(u.z) - 1.0);
    r[q] = p.r * (1.0 + sj * (2.0 * u01(u.w) - 1.0));
    gid[q] = (uint32_t)g;
}

// generate the rank's particles into caller-format device arrays (x: 3n, r: n, gid: n), allocated
// through alloc(bytes) (the context's allocator); n = 0 allowed
bool generate_bed(const dem_generator &g, const dem_box &box, double slab_lo, double slab_hi,
                  void *(*alloc)(size_t, void *), void *actx, cudaStream_t s, double **x, double **r, uint32_t **gid,
                  int64_t *n, std::string &err)
{
    std::vector<GenPlane> P;
    int64_t nl = 0;
    if (!build_planes(g, box, slab_lo, slab_hi, P, nl, err)) return false;
    *n = nl;
    *x = (double *)alloc(std::max<size_t>(8, 3 * nl * sizeof(double)), actx);
    *r = (double *)alloc(std::max<size_t>(8, nl * sizeof(double)), actx);
    *gid = (uint32_t *)alloc(std::max<size_t>(8, nl * sizeof(uint32_t)), actx);
    GenPlane *dP = (GenPlane *)alloc(std::max<size_t>(8, P.size() * sizeof(GenPlane)), actx);
    if (!*x || !*r || !*gid || !dP) { err = "generator: allocation failed"; return false; }
    if (nl) {
        cudaMemcpyAsync(dP, P.data(), P.size() * sizeof(GenPlane), cudaMemcpyHostToDevice, s);
        k_generate<<<(unsigned)((nl + 255) / 256), 256, 0, s>>>(nl, dP, (int)P.size(), g.seed, g.pos_jitter, g.size_jitter,
                                                              *x, *r, *gid);
    }
    if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) { err = "generator kernel failed"; return false; }
    return true;
}

extern "C" dem_status dem_generator_count(const dem_generator *gen, const dem_box *box, double slab_lo, double slab_hi,
                                          int64_t *n)
{
    if (!gen || !box || !n) return DEM_ERR_INVALID;
    std::vector<GenPlane> P;
    std::string err;
    int64_t nl = 0;
    if (!build_planes(*gen, *box, slab_lo, slab_hi, P, nl, err)) return DEM_ERR_INVALID;
    *n = nl;
    return DEM_OK;
}
