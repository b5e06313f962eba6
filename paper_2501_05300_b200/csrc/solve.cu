// solve.cu -- the nonsmooth contact solve and integration of one DEM step:
//
//  k_prepare    mass-splitting weights c/m, c/I per particle (c = contact count)
//  k_rows       impact trigger and Newton impact rows, SPOOK rows of the Hertz-mapped
//               normal constraint (reading R4)
//  (the Jacobi sweep itself is sweep.cu)
//  k_apply      gravity + warm-start impulses (MODE_APPLY) and per-particle force/torque
//               evaluation (MODE_FORCES), one thread per particle
//  k_integrate  x += h v, displacement since rebuild, KE / max|v| / NaN flags
//  k_plate_sum + k_boundary   int64 fixed-point plate reactions, plate drives, moving walls
#include "common.cuh"
#include "kernels.h"
#include "sweep_core.cuh"


__device__ __forceinline__ void boundary_vel(uint32_t p, const DevBoundary *__restrict__ bnd, d3 &v, double &mt)
{
    double mr;
    boundary_body(p, bnd, v, mt, mr);
}

__global__ void k_prepare(int64_t N, const uint32_t *__restrict__ inc_start, const double4 *__restrict__ pos,
                          double4 *__restrict__ vel, double4 *__restrict__ ang, double rho)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double c = (double)(inc_start[i + 1] - inc_start[i]);
    const double d = 2.0 * pos[i].w;
    const double m = rho * 3.14159265358979323846 * d * d * d / 6.0;
    const double I = m * d * d / 10.0;
    vel[i].w = c / m;
    ang[i].w = c / I;
}

// mode 0: impact trigger + impact rows into row_imp; mode 1: main SPOOK rows into row
__global__ void k_rows(int64_t nc, int mode, const uint2 *__restrict__ cij, const G4 *__restrict__ geo,
                       const double *__restrict__ cdel, R4 *__restrict__ row, R4 *__restrict__ row_imp,
                       const double4 *__restrict__ vel, const double4 *__restrict__ pos,
                       const DevBoundary *__restrict__ bnd, SolveParams sp, StepScalars *sc)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const uint2 ij = cij[c];
    const G4 g = geo[c];
    const d3 n = mk(g.x, g.y, g.z);
    const d3 va = xyz(vel[ij.x]);
    d3 vb;
    const bool ext = (ij.y & PARTNER_EXT) != 0;
    if (!ext) vb = xyz(vel[ij.y]);
    else { double mt; boundary_vel(ij.y, bnd, vb, mt); }
    const double un = dot(n, vb - va);
    R4 rw = row[c];
    if (mode == 0) {
        const bool imp = un < -sp.v_imp;
        if (imp) sc->impact = 1u;    // benign race: every writer stores 1
        row_imp[c] = mkR4(0, imp ? -sp.e_rest * un : 0.0, rw.z, rw.w);
        return;
    }
    // SPOOK: Sigma-hat = 4 Ups / (h^2 e_H k_n delta^(2 e_H - 2)), b = (4 Ups/h)(delta/e_H) + Ups u_n
    const double delta = cdel[c];
    const double ra = pos[ij.x].w;
    const double S = spook_sigma(sp, ext ? ra : rstar(ra, pos[ij.y].w), delta);
    row[c] = mkR4(S, 4.0 * sp.Ups / sp.h * (delta / sp.e_H) + sp.Ups * un, rw.z, rw.w);
}

// gravity + warm start (MODE_APPLY) or force/torque (MODE_FORCES, O6)
template <int MODE>
__global__ void k_apply(int64_t N, const double4 *__restrict__ vin, const double4 *__restrict__ win,
                        double4 *__restrict__ vout, double4 *__restrict__ wout, const uint32_t *__restrict__ inc_start,
                        const uint2 *__restrict__ inc, const G4 *__restrict__ geo, const R4 *__restrict__ row,
                        const P4 *__restrict__ Pa, const P4 *__restrict__ Pb, SolveParams sp)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t s = inc_start[i], e = inc_start[i + 1];
    d3 aL = mk(0, 0, 0), aA = mk(0, 0, 0);
    for (uint32_t k = s; k < e; k++) {
        const uint2 ent = inc[k];
        const uint32_t c = ent.x & INC_CMASK;
        const bool isB = (ent.x & B_SIDE) != 0;
        const G4 g = geo[c];
        const R4 rw = row[c];
        const P4 pa = Pa[c], pb = Pb[c];
        const d3 n = mk(g.x, g.y, g.z);
        const d3 Pt = mk(pa.y, pa.z, pa.w), Pr = mk(pb.x, pb.y, pb.z);
        const d3 L = (double)pa.x * n + Pt;
        const d3 nxPt = cross(n, Pt);
        if (isB) {
            aL = aL + L;
            aA = aA + ((-(double)rw.w) * nxPt + Pr);
        } else {
            aL = aL - L;
            aA = aA - ((double)rw.z * nxPt + Pr);
        }
    }
    if (MODE == SWEEP_MODE_FORCES) {
        const double ih = 1.0 / sp.h;
        vout[i] = make_double4(ih * aL.x, ih * aL.y, ih * aL.z, 0.0);
        wout[i] = make_double4(ih * aA.x, ih * aA.y, ih * aA.z, 0.0);
        return;
    }
    double4 V = vin[i], W = win[i];
    V.x += sp.h * sp.g[0];
    V.y += sp.h * sp.g[1];
    V.z += sp.h * sp.g[2];
    const uint32_t cnt = e - s;
    if (cnt) {
        const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
        V.x += im * aL.x; V.y += im * aL.y; V.z += im * aL.z;
        W.x += iI * aA.x; W.y += iI * aA.y; W.z += iI * aA.z;
    }
    vout[i] = V;
    wout[i] = W;
}

// x^{k+1} = x^k + h v^{k+1} + reductions for the report and the rebuild trigger
__global__ void k_integrate(int64_t N, const uint8_t *__restrict__ own, double4 *__restrict__ pos, const double4 *__restrict__ vel,
                            const double4 *__restrict__ ang, const double4 *__restrict__ xref, double h, double rho,
                            double *__restrict__ ke_part, StepScalars *sc)
{
    __shared__ double sk[256], sd[256], sv[256];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double ke = 0.0, disp = 0.0, vm = 0.0;
    if (i < N) {
        double4 p = pos[i];
        const double4 v = vel[i], w = ang[i];
        p.x = __dadd_rn(p.x, __dmul_rn(h, v.x));
        p.y = __dadd_rn(p.y, __dmul_rn(h, v.y));
        p.z = __dadd_rn(p.z, __dmul_rn(h, v.z));
        pos[i] = p;
        const double4 r = xref[i];
        const double dx = p.x - r.x, dy = p.y - r.y, dz = p.z - r.z;
        disp = sqrt(dx * dx + dy * dy + dz * dz);
        const double d = 2.0 * p.w;
        const double m = rho * 3.14159265358979323846 * d * d * d / 6.0, I = m * d * d / 10.0;
        const double v2 = v.x * v.x + v.y * v.y + v.z * v.z, w2 = w.x * w.x + w.y * w.y + w.z * w.z;
        ke = 0.5 * m * v2 + 0.5 * I * w2;
        vm = sqrt(v2);
        if (!isfinite(disp) || !isfinite(ke) || !isfinite(vm)) {
            atomicOr(&sc->nan_flag, 1u);
            disp = 0.0;
            ke = 0.0;
            vm = 0.0;
        }
        if (own && !own[i]) { disp = 0.0; ke = 0.0; vm = 0.0; }    // ghosts: reported by their owner
    }
    // block maxima first (non-negative doubles order like their bit patterns), one atomic per block
    sd[threadIdx.x] = disp;
    sv[threadIdx.x] = vm;
    sk[threadIdx.x] = ke;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sk[threadIdx.x] += sk[threadIdx.x + o];
            sd[threadIdx.x] = fmax(sd[threadIdx.x], sd[threadIdx.x + o]);
            sv[threadIdx.x] = fmax(sv[threadIdx.x], sv[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ke_part[blockIdx.x] = sk[0];
        atomicMax(&sc->max_disp_bits, (unsigned long long)__double_as_longlong(sd[0]));
        atomicMax(&sc->max_v_bits, (unsigned long long)__double_as_longlong(sv[0]));
    }
}

__global__ void k_reduce_ke(const double *__restrict__ part, int64_t nb, StepScalars *sc)
{
    __shared__ double sk[256];
    double s = 0.0;
    for (int64_t b = threadIdx.x; b < nb; b += 256) s += part[b];
    sk[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sk[threadIdx.x] += sk[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) sc->ke = sk[0];
}

// plate and wall reactions: F = (1/h) sum_{c on the body} (P_n n + P_t), int64 fixed point
// (order-free, exact; slots: plates 0..7, walls 8..13)
__global__ void k_plate_sum(int64_t nc, const uint8_t *__restrict__ own, const uint2 *__restrict__ cij, const G4 *__restrict__ geo,
                            const P4 *__restrict__ Pa, unsigned long long *__restrict__ acc,
                            unsigned int *__restrict__ pcount)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    if (own && !own[cij[c].x]) return;                   // a ghost's plate contact: its owner adds it
    const uint32_t j = cij[c].y;
    if (!(j & PARTNER_EXT)) return;
    const int q = (j & PARTNER_PLATE) ? (int)((j >> 4) & 0xF) : DEM_MAX_PLATES + (int)(j & ~PARTNER_EXT);
    const G4 g = geo[c];
    const P4 a = Pa[c];
    const double L[3] = {(double)a.x * g.x + a.y, (double)a.x * g.y + a.z, (double)a.x * g.z + a.w};
    for (int k = 0; k < 3; k++)
        atomicAdd(&acc[3 * q + k], (unsigned long long)llrint(L[k] * FIXED_SCALE));
    atomicAdd(&pcount[q], 1u);
}

// walls and plates advance with the velocity used in this step, then drives update the plate
// velocities for the next step (reading R18): kinematic ramp or staggered force axis
__global__ void k_boundary(DevBoundary *bnd, const unsigned long long *__restrict__ acc,
                           const unsigned int *__restrict__ pcount, double h, StepScalars *sc)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double disp = 0.0;
    for (int w = 0; w < 6; w++) {
        for (int k = 0; k < 3; k++) bnd->wp[w][k] = __dadd_rn(bnd->wp[w][k], __dmul_rn(__dmul_rn(h, bnd->wvel[w]), bnd->wn[w][k]));
        double d2 = 0.0;
        for (int k = 0; k < 3; k++) { const double d = bnd->wp[w][k] - bnd->wp_ref[w][k]; d2 += d * d; }
        disp = fmax(disp, sqrt(d2));
    }
    const double t1 = __dadd_rn(bnd->time, h);
    for (int w = 0; w < 6; w++) {
        for (int k = 0; k < 3; k++)
            bnd->wforce[w][k] = (double)(long long)acc[3 * (DEM_MAX_PLATES + w) + k] / FIXED_SCALE / h;
        bnd->wcount[w] = pcount[DEM_MAX_PLATES + w];
    }
    for (int q = 0; q < bnd->n_plates; q++) {
        for (int k = 0; k < 3; k++) {
            bnd->pforce[q][k] = (double)(long long)acc[3 * q + k] / FIXED_SCALE / h;
            bnd->ppos[q][k] = __dadd_rn(bnd->ppos[q][k], __dmul_rn(h, bnd->pvel[q][k]));
        }
        bnd->pcount[q] = pcount[q];
        for (int k = 0; k < 3; k++) {
            const int md = bnd->mode[q][k];
            const double v = bnd->pvel[q][k], fc = bnd->pforce[q][k], m = bnd->pmass[q];
            if (md == 2) {
                // staggered (R18); monolithic (R18b): the solve already set the velocity
                if (!bnd->mono) bnd->pvel[q][k] = v + h * (bnd->target[q][k] + fc) / m;
                bnd->pmotor[q][k] = bnd->target[q][k];
                continue;
            }
            double u1 = 0.0;   // locked axes: u = 0, never limited
            if (md == 1) {
                double s = bnd->ramp[q][k] > 0.0 ? (t1 - bnd->t0[q][k]) / bnd->ramp[q][k] : 1.0;
                s = s > 1.0 ? 1.0 : (s < 0.0 ? 0.0 : s);
                u1 = bnd->target[q][k] * s;
            }
            // staggered motor (reading R18 + Eq. 4): the force that brings the axis to u(t1)
            // against this step's contact reaction, clamped to [f_min, f_max]
            const double lam = m * (u1 - v) / h - fc;
            if (md == 1 && bnd->plimit[q][k] && (lam < bnd->pfmin[q][k] || lam > bnd->pfmax[q][k])) {
                const double lc = lam < bnd->pfmin[q][k] ? bnd->pfmin[q][k] : bnd->pfmax[q][k];
                bnd->pvel[q][k] = v + h * (lc + fc) / m;
                bnd->pmotor[q][k] = lc;
            } else {
                bnd->pvel[q][k] = u1;
                bnd->pmotor[q][k] = lam;
            }
        }
        double d2 = 0.0;
        for (int k = 0; k < 3; k++) { const double d = bnd->ppos[q][k] - bnd->ppos_ref[q][k]; d2 += d * d; }
        disp = fmax(disp, sqrt(d2));
    }
    bnd->time = t1;
    sc->bnd_disp = disp;
}

// ------------------------------------------------------------------ monolithic plates (R18b)
// owned plate contacts of the step (each contact counted once over the ranks)
__global__ void k_plate_flag(int64_t nc, const uint8_t *__restrict__ own, const uint2 *__restrict__ cij,
                             uint32_t *__restrict__ flag)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const uint32_t j = cij[c].y;
    flag[c] = ((j & (PARTNER_EXT | PARTNER_PLATE)) == (PARTNER_EXT | PARTNER_PLATE) && (!own || own[cij[c].x])) ? 1u : 0u;
}
// the impulse the plate received over a sweep: sum of (P_n n + P_t)(out) - (...)(in), int64 fixed
// point (exact, order-free); in == nullptr: the whole impulse of `out` (the warm start)
__global__ void k_plate_hub(int64_t n, const uint32_t *__restrict__ list, const uint2 *__restrict__ cij,
                            const G4 *__restrict__ geo, const void *__restrict__ pin, const void *__restrict__ pout,
                            unsigned long long *__restrict__ acc)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t c = list[t];
    const int q = (cij[c].y >> 4) & 0xF;
    const G4 g = geo[c];
    const P4 o = ((const P4 *)pout)[c];
    P4 i = mkP4(0, 0, 0, 0);
    if (pin) i = ((const P4 *)pin)[c];
    const double dPn = (double)o.x - (double)i.x;
    const double d[3] = {dPn * g.x + ((double)o.y - (double)i.y), dPn * g.y + ((double)o.z - (double)i.z),
                         dPn * g.z + ((double)o.w - (double)i.w)};
    for (int k = 0; k < 3; k++) atomicAdd(&acc[3 * q + k], (unsigned long long)llrint(d[k] * HUB_SCALE));
}
// force-driven axes take the increments (first: also the external impulse h F); acc is cleared
__global__ void k_plate_kick(DevBoundary *bnd, unsigned long long *acc, double h, int first)
{
    if (threadIdx.x || blockIdx.x) return;
    for (int q = 0; q < bnd->n_plates; q++)
        for (int k = 0; k < 3; k++) {
            const double dl = (double)(long long)acc[3 * q + k] / HUB_SCALE;
            acc[3 * q + k] = 0ull;
            if (bnd->mode[q][k] != 2) continue;
            bnd->pvel[q][k] += ((first ? h * bnd->target[q][k] : 0.0) + dl) / bnd->pmass[q];
        }
}
#define PGRID(n) (unsigned)(((n) + 255) / 256), 256, 0, s
void launch_plate_list_flags(int64_t nc, const uint8_t *own, const uint2 *cij, uint32_t *flag, cudaStream_t s)
{ if (nc) k_plate_flag<<<PGRID(nc)>>>(nc, own, cij, flag); }
void launch_plate_hub(int64_t n, const uint32_t *list, const uint2 *cij, const G4 *geo, const void *pin,
                      const void *pout, unsigned long long *acc, cudaStream_t s)
{
    if (!n) return;
    k_plate_hub<<<PGRID(n)>>>(n, list, cij, geo, pin, pout, acc);
}
void launch_plate_kick(DevBoundary *bnd, unsigned long long *acc, double h, int first, cudaStream_t s)
{ k_plate_kick<<<1, 32, 0, s>>>(bnd, acc, h, first); }
#undef PGRID

// step report: at the final velocities, per owned contact
// the normal complementarity residual |min(P_n, u_n + Sigma P_n - b)| and the cone excesses
// |P_t| - mu_t P_n, |P_r| - mu_r R* P_n (non-negative maxima as ordered double bits)
// grid-stride over the contacts, block maxima in shared memory, one atomic per block and
// quantity (a per-warp atomic on one address serialised 1.4 M updates at L2: 3.7 ms per launch)
__global__ void __launch_bounds__(256) k_residuals(int64_t nc, const uint8_t *__restrict__ own, const uint2 *__restrict__ cij,
                            const G4 *__restrict__ geo, const R4 *__restrict__ row, const double4 *__restrict__ vel,
                            const P4 *__restrict__ Pa, const P4 *__restrict__ Pb, const DevBoundary *__restrict__ bnd,
                            SolveParams sp, StepScalars *sc)
{
    __shared__ double sm[2][8];
    double res = 0.0, cone = 0.0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        const uint2 ij = cij[c];
        if (own && !own[ij.x]) continue;
        const G4 g = geo[c];
        const R4 rw = row[c];
        const P4 a = Pa[c], b = Pb[c];
        const d3 n = mk(g.x, g.y, g.z);
        d3 vb;
        double mt = sp.mu_t;
        if (!(ij.y & PARTNER_EXT)) vb = xyz(vel[ij.y]);
        else boundary_vel(ij.y, bnd, vb, mt);
        const double Pn = a.x;
        const double un = dot(n, vb - xyz(vel[ij.x]));
        const double wn = un + rw.x * Pn - rw.y;
        res = fmax(res, fabs(Pn < wn ? Pn : wn));
        const double e1 = sqrt((double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w) - mt * Pn;
        const double e2 = sqrt((double)b.x * b.x + (double)b.y * b.y + (double)b.z * b.z) - g.w * Pn;
        cone = fmax(cone, fmax(0.0, fmax(e1, e2)));
    }
    for (int o = 16; o; o >>= 1) {
        res = fmax(res, __shfl_xor_sync(0xffffffffu, res, o));
        cone = fmax(cone, __shfl_xor_sync(0xffffffffu, cone, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sm[0][w] = res; sm[1][w] = cone; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); q++) { res = fmax(res, sm[0][q]); cone = fmax(cone, sm[1][q]); }
        if (res > 0.0) atomicMax(&sc->max_res_bits, (unsigned long long)__double_as_longlong(res));
        if (cone > 0.0) atomicMax(&sc->max_cone_bits, (unsigned long long)__double_as_longlong(cone));
    }
}

__global__ void k_scatter_P(int64_t nc, const uint32_t *__restrict__ ccand, const P4 *__restrict__ Pa,
                            const P4 *__restrict__ Pb, P4 *__restrict__ Pca, P4 *__restrict__ Pcb)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    // back to candidate orientation (k_compact flipped the pair to canonical)
    const uint32_t kf = ccand[c], k = kf & ~CCAND_FLIP;
    P4 a = Pa[c], b = Pb[c];
    if (kf & CCAND_FLIP) { a.y = -a.y; a.z = -a.z; a.w = -a.w; b.x = -b.x; b.y = -b.y; b.z = -b.z; }
    Pca[k] = a;
    Pcb[k] = b;
}

// sorted order -> ascending-gid order (rank of gid in the sorted gid list)
__global__ void k_to_gid_order(int64_t N, const uint8_t *__restrict__ own, const uint32_t *__restrict__ gid, const uint32_t *__restrict__ gid_sorted,
                               const double4 *__restrict__ a, const double4 *__restrict__ b,
                               const double4 *__restrict__ c, double *__restrict__ oa, double *__restrict__ ob,
                               double *__restrict__ oc, double *__restrict__ orad, uint32_t *__restrict__ ogid, int64_t n_sorted)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N || (own && !own[i])) return;         // ghosts are reported by their owner
    const uint32_t gv = gid[i];
    int64_t lo = 0, hi = n_sorted;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (gid_sorted[mid] < gv) lo = mid + 1; else hi = mid;
    }
    const int64_t o = lo;
    if (oa) { const double4 v = a[i]; oa[3 * o] = v.x; oa[3 * o + 1] = v.y; oa[3 * o + 2] = v.z; }
    if (ob) { const double4 v = b[i]; ob[3 * o] = v.x; ob[3 * o + 1] = v.y; ob[3 * o + 2] = v.z; }
    if (oc) { const double4 v = c[i]; oc[3 * o] = v.x; oc[3 * o + 1] = v.y; oc[3 * o + 2] = v.z; }
    if (orad) orad[o] = a[i].w;
    if (ogid) ogid[o] = gv;
}

// keep particles with lo <= x[axis] <= hi: compaction of the gid-ordered export
__global__ void k_keep_flags(int64_t n, const double *__restrict__ x, int axis, double lo, double hi,
                             uint32_t *__restrict__ flag)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { const double v = x[3 * i + axis]; flag[i] = (v >= lo && v <= hi) ? 1u : 0u; }
}
__global__ void k_keep_gather(int64_t n, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ scan,
                              const double *__restrict__ x, const double *__restrict__ r, const double *__restrict__ v,
                              const double *__restrict__ w, const uint32_t *__restrict__ g, double *__restrict__ ox,
                              double *__restrict__ orr, double *__restrict__ ov, double *__restrict__ ow,
                              uint32_t *__restrict__ og)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !flag[i]) return;
    const uint32_t o = scan[i];
    for (int k = 0; k < 3; k++) { ox[3 * o + k] = x[3 * i + k]; ov[3 * o + k] = v[3 * i + k]; ow[3 * o + k] = w[3 * i + k]; }
    orr[o] = r[i];
    og[o] = g[i];
}
void launch_keep(int64_t n, const double *x, int axis, double lo, double hi, uint32_t *flag, cudaStream_t s)
{ if (n) k_keep_flags<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, x, axis, lo, hi, flag); }
void launch_keep_gather(int64_t n, const uint32_t *flag, const uint32_t *scan, const double *x, const double *r,
                        const double *v, const double *w, const uint32_t *g, double *ox, double *orr, double *ov,
                        double *ow, uint32_t *og, cudaStream_t s)
{ if (n) k_keep_gather<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, flag, scan, x, r, v, w, g, ox, orr, ov, ow, og); }

// caller arrays -> internal double4 layout
__global__ void k_load_state(int64_t N, const double *__restrict__ x, const double *__restrict__ r,
                             const double *__restrict__ v, const double *__restrict__ w,
                             const uint32_t *__restrict__ gid_in, double4 *__restrict__ pos,
                             double4 *__restrict__ vel, double4 *__restrict__ ang, uint32_t *__restrict__ gid)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    pos[i] = make_double4(x[3 * i], x[3 * i + 1], x[3 * i + 2], r[i]);
    vel[i] = v ? make_double4(v[3 * i], v[3 * i + 1], v[3 * i + 2], 0.0) : make_double4(0, 0, 0, 0);
    ang[i] = w ? make_double4(w[3 * i], w[3 * i + 1], w[3 * i + 2], 0.0) : make_double4(0, 0, 0, 0);
    gid[i] = gid_in ? gid_in[i] : (uint32_t)i;
}

// ------------------------------------------------------------------ launchers
#define GRID(n) (unsigned)(((n) + 255) / 256), 256, 0, s

void launch_prepare(int64_t N, const uint32_t *inc_start, const double4 *pos, double4 *vel, double4 *ang, double rho,
                    cudaStream_t s)
{ if (N) k_prepare<<<GRID(N)>>>(N, inc_start, pos, vel, ang, rho); }
void launch_rows(int64_t nc, int mode, const uint2 *cij, const G4 *geo, const double *cdel, R4 *row, R4 *row_imp,
                 const double4 *vel, const double4 *pos, const DevBoundary *bnd, const SolveParams &sp, StepScalars *sc,
                 cudaStream_t s)
{ if (nc) k_rows<<<GRID(nc)>>>(nc, mode, cij, geo, cdel, row, row_imp, vel, pos, bnd, sp, sc); }
// gravity + warm start (MODE_APPLY) or per-particle contact force/torque (MODE_FORCES)
void launch_apply(int mode, int64_t N, const double4 *vin, const double4 *win, double4 *vout, double4 *wout,
                  const uint32_t *inc_start, const uint2 *inc, const G4 *geo, const R4 *row, const P4 *Pa,
                  const P4 *Pb, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    if (mode == SWEEP_MODE_APPLY)
        k_apply<SWEEP_MODE_APPLY><<<GRID(N)>>>(N, vin, win, vout, wout, inc_start, inc, geo, row, Pa, Pb, sp);
    else
        k_apply<SWEEP_MODE_FORCES><<<GRID(N)>>>(N, vin, win, vout, wout, inc_start, inc, geo, row, Pa, Pb, sp);
}
void launch_integrate(int64_t N, const uint8_t *own, double4 *pos, const double4 *vel, const double4 *ang, const double4 *xref, double h,
                      double rho, double *ke_part, StepScalars *sc, cudaStream_t s)
{
    if (!N) return;
    const int64_t nb = (N + 255) / 256;
    k_integrate<<<GRID(N)>>>(N, own, pos, vel, ang, xref, h, rho, ke_part, sc);
    k_reduce_ke<<<1, 256, 0, s>>>(ke_part, nb, sc);
}
void launch_plate_sum(int64_t nc, const uint8_t *own, const uint2 *cij, const G4 *geo, const P4 *Pa, unsigned long long *acc,
                      unsigned int *pcount, cudaStream_t s)
{
    cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 3 * NB_SLOTS, s);
    cudaMemsetAsync(pcount, 0, sizeof(unsigned int) * NB_SLOTS, s);
    if (nc) k_plate_sum<<<GRID(nc)>>>(nc, own, cij, geo, Pa, acc, pcount);
}
void launch_boundary(DevBoundary *bnd, const unsigned long long *acc, const unsigned int *pcount, double h, StepScalars *sc,
                     cudaStream_t s)
{ k_boundary<<<1, 32, 0, s>>>(bnd, acc, pcount, h, sc); }
void launch_residuals(int64_t nc, const uint8_t *own, const uint2 *cij, const G4 *geo, const R4 *row, const double4 *vel,
                      const P4 *Pa, const P4 *Pb, const DevBoundary *bnd, const SolveParams &sp, StepScalars *sc,
                      cudaStream_t s)
{ if (nc) k_residuals<<<(unsigned)std::min<int64_t>((nc + 255) / 256, 148 * 8), 256, 0, s>>>(nc, own, cij, geo, row, vel, Pa, Pb, bnd, sp, sc); }
void launch_scatter_P(int64_t nc, const uint32_t *ccand, const P4 *Pa, const P4 *Pb, P4 *Pca, P4 *Pcb, cudaStream_t s)
{ if (nc) k_scatter_P<<<GRID(nc)>>>(nc, ccand, Pa, Pb, Pca, Pcb); }
void launch_to_gid_order(int64_t N, int64_t n_sorted, const uint8_t *own, const uint32_t *gid, const uint32_t *gid_sorted, const double4 *a,
                         const double4 *b, const double4 *c, double *oa, double *ob, double *oc, double *orad,
                         uint32_t *ogid, cudaStream_t s)
{ if (N) k_to_gid_order<<<GRID(N)>>>(N, own, gid, gid_sorted, a, b, c, oa, ob, oc, orad, ogid, n_sorted); }
void launch_load_state(int64_t N, const double *x, const double *r, const double *v, const double *w,
                       const uint32_t *gid_in, double4 *pos, double4 *vel, double4 *ang, uint32_t *gid, cudaStream_t s)
{ if (N) k_load_state<<<GRID(N)>>>(N, x, r, v, w, gid_in, pos, vel, ang, gid); }
