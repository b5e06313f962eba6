// sweep_core.cuh -- the contact-local projected impulse update (P:115-125 under SPOOK, P:132;
// readings R2, R4, R7-R10), shared by the Jacobi sweep (sweep.cu) and the coloured Gauss-Seidel
// sweep (gs.cu).
#pragma once
#include "common.cuh"

__device__ __forceinline__ d3 xyz(double4 a) { return mk(a.x, a.y, a.z); }

// factor that scales a vector of squared length m2 onto the ball of radius lim (1 inside):
// MUFU.RSQ64H estimate + one fp64 Newton step (1e-14), branch-free, full fp64 exponent range
__device__ __forceinline__ double clamp_scale(double m2, double lim)
{
    const bool out = m2 > lim * lim;
    const double q = out ? m2 : 1.0;
    return out ? lim * rsqrt64_1(q) : 1.0;
}

// value as stored (float or double impulse storage) and back as a double
template <typename T> __device__ __forceinline__ double rnd_st(double x, T &st)
{
    st = (T)x;
    return (double)st;
}

// Raw increments of one contact update: body a receives -(L), -(la n x dPt + dPr), body b
// receives +L, -lb n x dPt + dPr (n from a to b, lever arms l_a = la n, l_b = -lb n); the new
// impulses in their storage precision (TN: P_n, TT: P_t and P_r).
template <typename TN, typename TT>
struct ContactOutT {
    d3 L, nxdPt, dPr;
    TN pn;
    TT pt[3], pr[3];
};

// Contact (a, b) in the canonical orientation.  VA..WB are body a's and body b's states
// (.w = mass-splitting weights c/m, c/I); S = Sigma-hat, b = SPOOK bias (reading R4);
// mrRs = mu_r R*; Pn0, Pt0, Pr0 the sweep-start impulses (stored values).  Every evaluation of a
// contact (both tiles of a cross-tile pair, every rank holding it) passes the same canonical
// operands through this one function: bit-identical.
template <typename TN, typename TT>
__device__ __forceinline__ ContactOutT<TN, TT> contact_core_t(const double4 VA, const double4 WA, const double4 VB,
                                                              const double4 WB, double mt, const d3 n, double mrRs,
                                                              double S, double b, double la, double lb, double Pn0,
                                                              const d3 Pt0, const d3 Pr0, int rolling_dims)
{
    const double wA = VA.w, wtA = WA.w, wB = VB.w, wtB = WB.w;
    const double Dn = wA + wB;
    const double Dt = Dn + la * la * wtA + lb * lb * wtB;
    const double Dr = wtA + wtB;
    const d3 dv = xyz(VB) - xyz(VA);
    // 1. normal row (P:117 under SPOOK): P_n' = max(0, P_n - (u_n + S P_n - b)/(D_n + S)).
    //    Its velocity update is along n and drops out of the tangential projection below.
    ContactOutT<TN, TT> o;
    double Pn = Pn0 - (dot(n, dv) + S * Pn0 - b) * rcp64(Dn + S);
    Pn = rnd_st(Pn > 0.0 ? Pn : 0.0, o.pn);
    const double dPn = Pn - Pn0;
    // 2. friction (disc of radius mu_t P_n', maximum dissipation P:123-125):
    //    u = (v_b + w_b x l_b) - (v_a + w_a x l_a) = dv - (lb w_b + la w_a) x n
    const d3 oA = xyz(WA), oB = xyz(WB);
    const d3 u = dv - cross(lb * oB + la * oA, n);
    const d3 ut = u - dot(u, n) * n;
    d3 Pt = Pt0 - rcp64(Dt) * ut;
    Pt = clamp_scale(dot(Pt, Pt), mt * Pn) * Pt;
    const d3 dPt = mk(rnd_st(Pt.x, o.pt[0]), rnd_st(Pt.y, o.pt[1]), rnd_st(Pt.z, o.pt[2])) - Pt0;
    o.nxdPt = cross(n, dPt);
    // 3. rolling (ball of radius mu_r R* P_n', readings R7/R8) on the spins updated by
    //    the friction increment: w_b - w_a + (wtA la - wtB lb) n x dPt
    d3 ur = (oB - oA) + (wtA * la - wtB * lb) * o.nxdPt;
    if (rolling_dims == 2) ur = ur - dot(ur, n) * n;
    d3 Pr = Pr0 - rcp64(Dr) * ur;
    Pr = clamp_scale(dot(Pr, Pr), mrRs * Pn) * Pr;
    o.dPr = mk(rnd_st(Pr.x, o.pr[0]), rnd_st(Pr.y, o.pr[1]), rnd_st(Pr.z, o.pr[2])) - Pr0;
    o.L = dPn * n + dPt;
    return o;
}

// fp32-impulse interface (P4 = float4 records: the coloured Gauss-Seidel sweep, gs.cu)
struct ContactOut {
    d3 L, nxdPt, dPr;
    P4 Pa, Pb;       // new impulses (P_n, P_t) / (P_r, 0)
};
__device__ __forceinline__ ContactOut contact_core(const double4 VA, const double4 WA, const double4 VB,
                                                   const double4 WB, double mt, const d3 n, double mrRs, double S,
                                                   double b, double la, double lb, const P4 pa, const P4 pb,
                                                   int rolling_dims)
{
    const ContactOutT<float, float> r = contact_core_t<float, float>(
        VA, WA, VB, WB, mt, n, mrRs, S, b, la, lb, (double)pa.x, mk(pa.y, pa.z, pa.w), mk(pb.x, pb.y, pb.z),
        rolling_dims);
    ContactOut o;
    o.L = r.L;
    o.nxdPt = r.nxdPt;
    o.dPr = r.dPr;
    o.Pa = make_float4(r.pn, r.pt[0], r.pt[1], r.pt[2]);
    o.Pb = make_float4(r.pr[0], r.pr[1], r.pr[2], 0.0f);
    return o;
}

// velocity of a boundary body at the contact (walls: along their normal; plates: translation)
// and the partner's friction coefficients
__device__ __forceinline__ void boundary_body(uint32_t p, const DevBoundary *__restrict__ bnd, d3 &v, double &mt,
                                              double &mr)
{
    const uint32_t code = p & ~PARTNER_EXT;
    if (code & PARTNER_PLATE) {
        const int q = (code >> 4) & 0xF;
        v = mk(bnd->pvel[q][0], bnd->pvel[q][1], bnd->pvel[q][2]);
        mt = bnd->pmu_t[q];
        mr = bnd->pmu_r[q];
    } else {
        const int w = (int)code;
        const double s = bnd->wvel[w];
        v = mk(s * bnd->wn[w][0], s * bnd->wn[w][1], s * bnd->wn[w][2]);
        mt = bnd->wall_mu_t;
        mr = bnd->wall_mu_r;
    }
}
