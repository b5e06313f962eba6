// solve.cu -- the nonsmooth contact solve and integration of one DEM step:
//
//  k_prepare    mass-splitting weights c/m, c/I per particle (c = contact count)
//  k_rows       impact trigger and Newton impact rows, SPOOK rows of the Hertz-mapped
//               normal constraint (reading R4)
//  k_sweep_tile one Jacobi projected-impulse sweep (P:134 solver run as Jacobi, reading R2).
//               A block owns a tile of TP consecutive (Morton-ordered) particles; its threads
//               walk the tile's half-contacts in chunks of TP (one half-contact per thread, all
//               lanes busy whatever the contact counts), recompute each incident contact from the
//               sweep-start velocities in the canonical (a, b) orientation -- bit-identical from
//               both ends -- and the owning particle sums its chunk contributions from shared
//               memory in CSR order: a deterministic segmented reduction, no float atomics.
//               Body a of a contact writes the new impulse (ping-pong buffers).
//  k_apply      gravity + warm-start impulses (MODE_APPLY) and per-particle force/torque
//               evaluation (MODE_FORCES), one thread per particle
//  k_integrate  x += h v, displacement since rebuild, KE / max|v| / NaN flags
//  k_plate_sum + k_boundary   int64 fixed-point plate reactions, plate drives, moving walls
#include "common.cuh"
#include "kernels.h"

__device__ __forceinline__ d3 xyz(double4 a) { return mk(a.x, a.y, a.z); }

// fp64 reciprocal: fp32 estimate + two Newton steps (relative error ~1e-16; operands are
// positive, finite and inside the fp32 range: split weights, regularised diagonals)
__device__ __forceinline__ double rcp64(double x)
{
    double r = (double)__frcp_rn((float)x);
    r = r * (2.0 - x * r);
    r = r * (2.0 - x * r);
    return r;
}

__device__ __forceinline__ void boundary_vel(uint32_t p, const DevBoundary *__restrict__ bnd, d3 &v, double &mt)
{
    const uint32_t code = p & ~PARTNER_EXT;
    if (code & PARTNER_PLATE) {
        const int q = (code >> 4) & 0xF;
        v = mk(bnd->pvel[q][0], bnd->pvel[q][1], bnd->pvel[q][2]);
        mt = bnd->pmu_t[q];
    } else {
        const int w = (int)code;
        const double s = bnd->wvel[w];
        v = mk(s * bnd->wn[w][0], s * bnd->wn[w][1], s * bnd->wn[w][2]);
        mt = bnd->wall_mu_t;
    }
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
    double S;
    if (sp.hertz) {
        const double ra = pos[ij.x].w;
        const double Rs = ext ? ra : ra * pos[ij.y].w / (ra + pos[ij.y].w);
        const double kn = sp.Es * sqrt(2.0 * Rs) / 3.0;        // k_n = E* sqrt(d*)/3, d* = 2 R*
        S = 4.0 * sp.Ups / (sp.h * sp.h * sp.e_H * kn * sqrt(delta));
    } else {
        S = 4.0 * sp.Ups / (sp.h * sp.h * sp.e_H * sp.k_lin);
    }
    row[c] = mkR4(S, 4.0 * sp.Ups / sp.h * (delta / sp.e_H) + sp.Ups * un, rw.z, rw.w);
}

// ------------------------------------------------------------------ the Jacobi sweep
// One half-contact: contact c seen from `self`.  Canonical orientation: a = cij.x, b = cij.y.
// Returns the contribution to self (dL linear, dA angular impulse) and the new impulse.
struct HalfOut {
    d3 dL, dA;
    P4 Pa, Pb;
};

__device__ __forceinline__ HalfOut half_contact(const double4 VS, const double4 WS, const double4 VP, const double4 WP,
                                                bool isB, double mt, const G4 g, const R4 rw, const P4 pa,
                                                const P4 pb, int rolling_dims)
{
    // canonical a/b by selects: one instruction stream for both ends -> bit-identical result
    const double4 VA = isB ? VP : VS, WA = isB ? WP : WS;
    const double4 VB = isB ? VS : VP, WB = isB ? WS : WP;
    const d3 n = mk(g.x, g.y, g.z);
    const double mrRs = g.w;                     // mu_r R*
    const double la = rw.z, lb = rw.w;           // lever arms l_a = la n, l_b = -lb n
    const double wA = VA.w, wtA = WA.w, wB = VB.w, wtB = WB.w;
    const double Dn = wA + wB;
    const double Dt = Dn + la * la * wtA + lb * lb * wtB;
    const double Dr = wtA + wtB;
    const d3 dv = xyz(VB) - xyz(VA);
    // 1. normal row (P:117 under SPOOK): P_n' = max(0, P_n - (u_n + S P_n - b)/(D_n + S)).
    //    Its velocity update is along n and drops out of the tangential projection below.
    const double S = rw.x, b = rw.y, Pn0 = pa.x;
    double Pn = Pn0 - (dot(n, dv) + S * Pn0 - b) * rcp64(Dn + S);
    Pn = rndP(Pn > 0.0 ? Pn : 0.0);
    const double dPn = Pn - Pn0;
    // 2. friction (disc of radius mu_t P_n', maximum dissipation P:123-125):
    //    u = (v_b + w_b x l_b) - (v_a + w_a x l_a) = dv - (lb w_b + la w_a) x n
    const d3 oA = xyz(WA), oB = xyz(WB);
    const d3 u = dv - cross(lb * oB + la * oA, n);
    const d3 ut = u - dot(u, n) * n;
    const d3 Pt0 = mk(pa.y, pa.z, pa.w);
    d3 Pt = Pt0 - rcp64(Dt) * ut;
    double lim = mt * Pn, m2 = dot(Pt, Pt);
    if (m2 > lim * lim) Pt = (lim * rsqrt(m2)) * Pt;
    const P4 PaN = mkP4(Pn, Pt.x, Pt.y, Pt.z);
    const d3 dPt = mk(PaN.y, PaN.z, PaN.w) - Pt0;
    const d3 nxdPt = cross(n, dPt);
    // 3. rolling (ball of radius mu_r R* P_n', readings R7/R8) on the spins updated by
    //    the friction increment: w_b - w_a + (wtA la - wtB lb) n x dPt
    d3 ur = (oB - oA) + (wtA * la - wtB * lb) * nxdPt;
    if (rolling_dims == 2) ur = ur - dot(ur, n) * n;
    const d3 Pr0 = mk(pb.x, pb.y, pb.z);
    d3 Pr = Pr0 - rcp64(Dr) * ur;
    lim = mrRs * Pn;
    m2 = dot(Pr, Pr);
    if (m2 > lim * lim) Pr = (lim * rsqrt(m2)) * Pr;
    const P4 PbN = mkP4(Pr.x, Pr.y, Pr.z, 0);
    const d3 dPr = mk(PbN.x, PbN.y, PbN.z) - Pr0;
    // 4. contribution to self: a gets -(dPn n + dPt), -(la n x dPt + dPr);
    //                          b gets +(dPn n + dPt), -lb n x dPt + dPr
    HalfOut o;
    const d3 L = dPn * n + dPt;
    o.dL = isB ? L : mk(-L.x, -L.y, -L.z);
    o.dA = isB ? ((-lb) * nxdPt + dPr) : mk(-(la * nxdPt.x + dPr.x), -(la * nxdPt.y + dPr.y), -(la * nxdPt.z + dPr.z));
    o.Pa = PaN;
    o.Pb = PbN;
    return o;
}

constexpr int TP = 128;

__global__ void __launch_bounds__(TP) k_sweep_tile(int64_t N, const double4 *__restrict__ vin,
                                                   const double4 *__restrict__ win, double4 *__restrict__ vout,
                                                   double4 *__restrict__ wout, const uint32_t *__restrict__ inc_start,
                                                   const uint2 *__restrict__ inc, const G4 *__restrict__ geo,
                                                   const R4 *__restrict__ row, const P4 *__restrict__ Pa_in,
                                                   const P4 *__restrict__ Pb_in, P4 *__restrict__ Pa_out,
                                                   P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd,
                                                   SolveParams sp)
{
    __shared__ double4 sV[TP], sW[TP];
    __shared__ uint32_t sI[TP + 1];
    __shared__ d3 sL[TP], sA[TP];
    const int t = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * TP;
    const int np = (int)min((int64_t)TP, N - p0);
    double4 V = make_double4(0, 0, 0, 0), W = V;
    if (t < np) {
        V = vin[p0 + t];
        W = win[p0 + t];
        sV[t] = V;
        sW[t] = W;
    }
    for (int q = t; q <= np; q += TP) sI[q] = inc_start[p0 + q];
    __syncthreads();
    uint32_t s_i = 0, e_i = 0;
    if (t < np) { s_i = sI[t]; e_i = sI[t + 1]; }
    const uint32_t k0 = sI[0], k1 = sI[np];
    d3 aL = mk(0, 0, 0), aA = mk(0, 0, 0);
    for (uint32_t kb = k0; kb < k1; kb += TP) {
        const uint32_t k = kb + t;
        if (k < k1) {
            int lo = 0, hi = np;                       // owner: sI[lo] <= k < sI[lo + 1]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (sI[mid] <= k) lo = mid; else hi = mid;
            }
            const uint2 ent = inc[k];
            const uint32_t c = ent.x & ~B_SIDE;
            const bool isB = (ent.x & B_SIDE) != 0;
            const uint32_t p = ent.y;
            double4 VP, WP;
            double mt;
            if (!(p & PARTNER_EXT)) {
                const int64_t pl = (int64_t)p - p0;
                if (pl >= 0 && pl < np) { VP = sV[pl]; WP = sW[pl]; }
                else { VP = vin[p]; WP = win[p]; }
                mt = sp.mu_t;
            } else {
                d3 bv;
                boundary_vel(p, bnd, bv, mt);
                VP = make_double4(bv.x, bv.y, bv.z, 0.0);
                WP = make_double4(0.0, 0.0, 0.0, 0.0);
            }
            const HalfOut o = half_contact(sV[lo], sW[lo], VP, WP, isB, mt, geo[c], row[c], Pa_in[c], Pb_in[c],
                                           sp.rolling_dims);
            if (!isB) {
                Pa_out[c] = o.Pa;
                Pb_out[c] = o.Pb;
            }
            sL[t] = o.dL;
            sA[t] = o.dA;
        }
        __syncthreads();
        if (t < np) {
            const uint32_t a = max(s_i, kb), b = min(e_i, kb + TP);
            for (uint32_t q = a; q < b; q++) {
                aL = aL + sL[q - kb];
                aA = aA + sA[q - kb];
            }
        }
        __syncthreads();
    }
    if (t < np) {
        // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
        const uint32_t cnt = e_i - s_i;
        if (cnt) {
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            V.x += im * aL.x; V.y += im * aL.y; V.z += im * aL.z;
            W.x += iI * aA.x; W.y += iI * aA.y; W.z += iI * aA.z;
        }
        vout[p0 + t] = V;
        wout[p0 + t] = W;
    }
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
        const uint32_t c = ent.x & ~B_SIDE;
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
__global__ void k_integrate(int64_t N, double4 *__restrict__ pos, const double4 *__restrict__ vel,
                            const double4 *__restrict__ ang, const double4 *__restrict__ xref, double h, double rho,
                            double *__restrict__ ke_part, StepScalars *sc)
{
    __shared__ double sk[256];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double ke = 0.0;
    if (i < N) {
        double4 p = pos[i];
        const double4 v = vel[i], w = ang[i];
        p.x = __dadd_rn(p.x, __dmul_rn(h, v.x));
        p.y = __dadd_rn(p.y, __dmul_rn(h, v.y));
        p.z = __dadd_rn(p.z, __dmul_rn(h, v.z));
        pos[i] = p;
        const double4 r = xref[i];
        const double dx = p.x - r.x, dy = p.y - r.y, dz = p.z - r.z;
        double disp = sqrt(dx * dx + dy * dy + dz * dz);
        const double d = 2.0 * p.w;
        const double m = rho * 3.14159265358979323846 * d * d * d / 6.0, I = m * d * d / 10.0;
        const double v2 = v.x * v.x + v.y * v.y + v.z * v.z, w2 = w.x * w.x + w.y * w.y + w.z * w.z;
        ke = 0.5 * m * v2 + 0.5 * I * w2;
        const double vm = sqrt(v2);
        if (!isfinite(disp) || !isfinite(ke)) {
            atomicOr(&sc->nan_flag, 1u);
            disp = 0.0;
            ke = 0.0;
        } else {
            atomicMax(&sc->max_disp_bits, (unsigned long long)__double_as_longlong(disp));
            atomicMax(&sc->max_v_bits, (unsigned long long)__double_as_longlong(vm));
        }
    }
    sk[threadIdx.x] = ke;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sk[threadIdx.x] += sk[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) ke_part[blockIdx.x] = sk[0];
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

// plate reaction: F_p = (1/h) sum_{c in p} (P_n n + P_t), int64 fixed point (order-free, exact)
__global__ void k_plate_sum(int64_t nc, const uint2 *__restrict__ cij, const G4 *__restrict__ geo,
                            const P4 *__restrict__ Pa, unsigned long long *__restrict__ acc,
                            unsigned int *__restrict__ pcount)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const uint32_t j = cij[c].y;
    if ((j & (PARTNER_EXT | PARTNER_PLATE)) != (PARTNER_EXT | PARTNER_PLATE)) return;
    const int q = (j >> 4) & 0xF;
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
    for (int q = 0; q < bnd->n_plates; q++) {
        for (int k = 0; k < 3; k++) {
            bnd->pforce[q][k] = (double)(long long)acc[3 * q + k] / FIXED_SCALE / h;
            bnd->ppos[q][k] = __dadd_rn(bnd->ppos[q][k], __dmul_rn(h, bnd->pvel[q][k]));
        }
        bnd->pcount[q] = pcount[q];
        for (int k = 0; k < 3; k++) {
            const int md = bnd->mode[q][k];
            if (md == 0) bnd->pvel[q][k] = 0.0;
            else if (md == 1) {
                double s = bnd->ramp[q][k] > 0.0 ? (t1 - bnd->t0[q][k]) / bnd->ramp[q][k] : 1.0;
                s = s > 1.0 ? 1.0 : (s < 0.0 ? 0.0 : s);
                bnd->pvel[q][k] = bnd->target[q][k] * s;
            } else {
                bnd->pvel[q][k] += h * (bnd->target[q][k] + bnd->pforce[q][k]) / bnd->pmass[q];
            }
        }
        double d2 = 0.0;
        for (int k = 0; k < 3; k++) { const double d = bnd->ppos[q][k] - bnd->ppos_ref[q][k]; d2 += d * d; }
        disp = fmax(disp, sqrt(d2));
    }
    bnd->time = t1;
    sc->bnd_disp = disp;
}

__global__ void k_scatter_P(int64_t nc, const uint32_t *__restrict__ ccand, const P4 *__restrict__ Pa,
                            const P4 *__restrict__ Pb, P4 *__restrict__ Pca, P4 *__restrict__ Pcb)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const uint32_t k = ccand[c];
    Pca[k] = Pa[c];
    Pcb[k] = Pb[c];
}

// sorted order -> ascending-gid order (rank of gid in the sorted gid list)
__global__ void k_to_gid_order(int64_t N, const uint32_t *__restrict__ gid, const uint32_t *__restrict__ gid_sorted,
                               const double4 *__restrict__ a, const double4 *__restrict__ b,
                               const double4 *__restrict__ c, double *__restrict__ oa, double *__restrict__ ob,
                               double *__restrict__ oc, double *__restrict__ orad, uint32_t *__restrict__ ogid)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t gv = gid[i];
    int64_t lo = 0, hi = N;
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
void launch_sweep(int mode, int64_t N, const double4 *vin, const double4 *win, double4 *vout, double4 *wout,
                  const uint32_t *inc_start, const uint2 *inc, const G4 *geo, const R4 *row,
                  const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out,
                  const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    if (mode == SWEEP_MODE_SWEEP)
        k_sweep_tile<<<(unsigned)((N + TP - 1) / TP), TP, 0, s>>>(N, vin, win, vout, wout, inc_start, inc, geo, row,
                                                                  Pa_in, Pb_in, Pa_out, Pb_out, bnd, sp);
    else if (mode == SWEEP_MODE_APPLY)
        k_apply<SWEEP_MODE_APPLY><<<GRID(N)>>>(N, vin, win, vout, wout, inc_start, inc, geo, row, Pa_in, Pb_in, sp);
    else
        k_apply<SWEEP_MODE_FORCES><<<GRID(N)>>>(N, vin, win, vout, wout, inc_start, inc, geo, row, Pa_in, Pb_in, sp);
}
void launch_integrate(int64_t N, double4 *pos, const double4 *vel, const double4 *ang, const double4 *xref, double h,
                      double rho, double *ke_part, StepScalars *sc, cudaStream_t s)
{
    if (!N) return;
    const int64_t nb = (N + 255) / 256;
    k_integrate<<<GRID(N)>>>(N, pos, vel, ang, xref, h, rho, ke_part, sc);
    k_reduce_ke<<<1, 256, 0, s>>>(ke_part, nb, sc);
}
void launch_plates(int64_t nc, const uint2 *cij, const G4 *geo, const P4 *Pa, unsigned long long *acc,
                   unsigned int *pcount, DevBoundary *bnd, double h, StepScalars *sc, cudaStream_t s)
{
    cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 3 * DEM_MAX_PLATES, s);
    cudaMemsetAsync(pcount, 0, sizeof(unsigned int) * DEM_MAX_PLATES, s);
    if (nc) k_plate_sum<<<GRID(nc)>>>(nc, cij, geo, Pa, acc, pcount);
    k_boundary<<<1, 32, 0, s>>>(bnd, acc, pcount, h, sc);
}
void launch_scatter_P(int64_t nc, const uint32_t *ccand, const P4 *Pa, const P4 *Pb, P4 *Pca, P4 *Pcb, cudaStream_t s)
{ if (nc) k_scatter_P<<<GRID(nc)>>>(nc, ccand, Pa, Pb, Pca, Pcb); }
void launch_to_gid_order(int64_t N, const uint32_t *gid, const uint32_t *gid_sorted, const double4 *a,
                         const double4 *b, const double4 *c, double *oa, double *ob, double *oc, double *orad,
                         uint32_t *ogid, cudaStream_t s)
{ if (N) k_to_gid_order<<<GRID(N)>>>(N, gid, gid_sorted, a, b, c, oa, ob, oc, orad, ogid); }
void launch_load_state(int64_t N, const double *x, const double *r, const double *v, const double *w,
                       const uint32_t *gid_in, double4 *pos, double4 *vel, double4 *ang, uint32_t *gid, cudaStream_t s)
{ if (N) k_load_state<<<GRID(N)>>>(N, x, r, v, w, gid_in, pos, vel, ang, gid); }
