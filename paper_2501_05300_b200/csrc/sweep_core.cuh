// sweep_core.cuh -- the contact-local projected impulse update of one Jacobi sweep (P:115-125
// under SPOOK; readings R2, R4, R7-R10), shared by every sweep kernel of libdem.so.
#pragma once
#include "common.cuh"

__device__ __forceinline__ d3 xyz(double4 a) { return mk(a.x, a.y, a.z); }

// factor that scales a vector of squared length m2 onto the ball of radius lim (1 inside):
// MUFU.RSQ64H estimate + two fp64 Newton steps, branch-free, full fp64 exponent range
__device__ __forceinline__ double clamp_scale(double m2, double lim)
{
    const bool out = m2 > lim * lim;
    const double q = out ? m2 : 1.0;
    return out ? lim * rsqrt64(q) : 1.0;
}

struct HalfOut {
    d3 dL, dA;       // contribution to `self` (linear, angular impulse)
    P4 Pa, Pb;       // new impulses (P_n, P_t) / (P_r, 0)
};

// Raw increments of one contact update: body a receives -(L), -(la n x dPt + dPr), body b
// receives +L, -lb n x dPt + dPr (n from a to b, lever arms l_a = la n, l_b = -lb n).
struct ContactOut {
    d3 L, nxdPt, dPr;
    P4 Pa, Pb;       // new impulses (P_n, P_t) / (P_r, 0)
};

#ifdef DEM_F32MATH
// Experimental (precision study): the projected update in fp32 arithmetic.  The
// cancelling differences (v_b - v_a, lever-arm spin sums, w_b - w_a) are formed in fp64 first;
// impulses are fp32 storage anyway; increments are returned in fp64 for the fp64 accumulation.
struct f3 { float x, y, z; };
__device__ __forceinline__ f3 f3m(float x, float y, float z) { return f3{x, y, z}; }
__device__ __forceinline__ f3 operator+(f3 a, f3 b) { return f3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ f3 operator-(f3 a, f3 b) { return f3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ f3 operator*(float s, f3 a) { return f3{s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ float dotf(f3 a, f3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ f3 crossf(f3 a, f3 b) { return f3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
__device__ __forceinline__ f3 tof(d3 a) { return f3{(float)a.x, (float)a.y, (float)a.z}; }
__device__ __forceinline__ d3 tod(f3 a) { return d3{(double)a.x, (double)a.y, (double)a.z}; }
__device__ __forceinline__ float rcpf(float x) { float r = __frcp_rn(x); return r; }
__device__ __forceinline__ float clampf(float m2, float lim) { return m2 > lim * lim ? lim * rsqrtf(m2) : 1.0f; }

__device__ __forceinline__ ContactOut contact_core(const double4 VA, const double4 WA, const double4 VB,
                                                   const double4 WB, double mt_, const d3 n_, double mrRs_, double S_,
                                                   double b_, double la_, double lb_, const P4 pa, const P4 pb,
                                                   int rolling_dims)
{
    const f3 n = tof(n_);
    const float la = (float)la_, lb = (float)lb_, S = (float)S_, b = (float)b_, mt = (float)mt_, mrRs = (float)mrRs_;
    const float wA = (float)VA.w, wtA = (float)WA.w, wB = (float)VB.w, wtB = (float)WB.w;
    const float Dn = wA + wB;
    const float Dt = Dn + la * la * wtA + lb * lb * wtB;
    const float Dr = wtA + wtB;
    const f3 dv = tof(xyz(VB) - xyz(VA));
    const f3 lw = tof(lb_ * xyz(WB) + la_ * xyz(WA));
    const f3 dw = tof(xyz(WB) - xyz(WA));
    ContactOut o;
    const float Pn0 = pa.x;
    float Pn = Pn0 - (dotf(n, dv) + S * Pn0 - b) * rcpf(Dn + S);
    Pn = Pn > 0.0f ? Pn : 0.0f;
    o.Pa.x = Pn;
    const f3 u = dv - crossf(lw, n);
    const f3 ut = u - dotf(u, n) * n;
    const f3 Pt0 = f3m(pa.y, pa.z, pa.w);
    f3 Pt = Pt0 - rcpf(Dt) * ut;
    Pt = clampf(dotf(Pt, Pt), mt * Pn) * Pt;
    o.Pa.y = Pt.x; o.Pa.z = Pt.y; o.Pa.w = Pt.z;
    const f3 dPt = Pt - Pt0;
    const f3 nxdPt = crossf(n, dPt);
    f3 ur = dw + (wtA * la - wtB * lb) * nxdPt;
    if (rolling_dims == 2) ur = ur - dotf(ur, n) * n;
    const f3 Pr0 = f3m(pb.x, pb.y, pb.z);
    f3 Pr = Pr0 - rcpf(Dr) * ur;
    Pr = clampf(dotf(Pr, Pr), mrRs * Pn) * Pr;
    o.Pb.x = Pr.x; o.Pb.y = Pr.y; o.Pb.z = Pr.z; o.Pb.w = 0.0f;
    // increments from the stored (fp32) impulses, exact in fp64
    const double dPn = (double)Pn - (double)Pn0;
    const d3 dPtd = d3{(double)Pt.x - (double)Pt0.x, (double)Pt.y - (double)Pt0.y, (double)Pt.z - (double)Pt0.z};
    o.nxdPt = cross(n_, dPtd);
    o.dPr = d3{(double)Pr.x - (double)Pr0.x, (double)Pr.y - (double)Pr0.y, (double)Pr.z - (double)Pr0.z};
    o.L = dPn * n_ + dPtd;
    return o;
}
#else
// Contact (a, b) in the canonical orientation.  VA..WB are body a's and body b's states
// (.w = mass-splitting weights c/m, c/I); S = Sigma-hat, b = SPOOK bias (reading R4);
// mrRs = mu_r R*.  Every kernel that evaluates a contact from both ends passes the same
// canonical operands through this one function, so both ends get bit-identical impulses.
__device__ __forceinline__ ContactOut contact_core(const double4 VA, const double4 WA, const double4 VB,
                                                   const double4 WB, double mt, const d3 n, double mrRs, double S,
                                                   double b, double la, double lb, const P4 pa, const P4 pb,
                                                   int rolling_dims)
{
    const double wA = VA.w, wtA = WA.w, wB = VB.w, wtB = WB.w;
    const double Dn = wA + wB;
    const double Dt = Dn + la * la * wtA + lb * lb * wtB;
    const double Dr = wtA + wtB;
    const d3 dv = xyz(VB) - xyz(VA);
    // 1. normal row (P:117 under SPOOK): P_n' = max(0, P_n - (u_n + S P_n - b)/(D_n + S)).
    //    Its velocity update is along n and drops out of the tangential projection below.
    ContactOut o;
    const double Pn0 = p_ld(pa.x);
    double Pn = Pn0 - (dot(n, dv) + S * Pn0 - b) * rcp64(Dn + S);
    Pn = p_rnd(Pn > 0.0 ? Pn : 0.0, o.Pa.x);
    const double dPn = Pn - Pn0;
    // 2. friction (disc of radius mu_t P_n', maximum dissipation P:123-125):
    //    u = (v_b + w_b x l_b) - (v_a + w_a x l_a) = dv - (lb w_b + la w_a) x n
    const d3 oA = xyz(WA), oB = xyz(WB);
    const d3 u = dv - cross(lb * oB + la * oA, n);
    const d3 ut = u - dot(u, n) * n;
    const d3 Pt0 = mk(p_ld(pa.y), p_ld(pa.z), p_ld(pa.w));
    d3 Pt = Pt0 - rcp64(Dt) * ut;
    Pt = clamp_scale(dot(Pt, Pt), mt * Pn) * Pt;
    const d3 dPt = mk(p_rnd(Pt.x, o.Pa.y), p_rnd(Pt.y, o.Pa.z), p_rnd(Pt.z, o.Pa.w)) - Pt0;
    o.nxdPt = cross(n, dPt);
    // 3. rolling (ball of radius mu_r R* P_n', readings R7/R8) on the spins updated by
    //    the friction increment: w_b - w_a + (wtA la - wtB lb) n x dPt
    d3 ur = (oB - oA) + (wtA * la - wtB * lb) * o.nxdPt;
    if (rolling_dims == 2) ur = ur - dot(ur, n) * n;
    const d3 Pr0 = mk(p_ld(pb.x), p_ld(pb.y), p_ld(pb.z));
    d3 Pr = Pr0 - rcp64(Dr) * ur;
    Pr = clamp_scale(dot(Pr, Pr), mrRs * Pn) * Pr;
    o.Pb.w = 0;
    o.dPr = mk(p_rnd(Pr.x, o.Pb.x), p_rnd(Pr.y, o.Pb.y), p_rnd(Pr.z, o.Pb.z)) - Pr0;
    o.L = dPn * n + dPt;
    return o;
}
#endif

// One half-contact: contact (a, b) seen from self (isB: self is body b).
__device__ __forceinline__ HalfOut half_core(const double4 VA, const double4 WA, const double4 VB, const double4 WB,
                                             bool isB, double mt, const d3 n, double mrRs, double S, double b,
                                             double la, double lb, const P4 pa, const P4 pb, int rolling_dims)
{
    const ContactOut c = contact_core(VA, WA, VB, WB, mt, n, mrRs, S, b, la, lb, pa, pb, rolling_dims);
    // contribution to self: a gets -(dPn n + dPt), -(la n x dPt + dPr);
    //                       b gets +(dPn n + dPt), -lb n x dPt + dPr
    HalfOut o;
    o.dL = isB ? c.L : mk(-c.L.x, -c.L.y, -c.L.z);
    o.dA = isB ? ((-lb) * c.nxdPt + c.dPr)
               : mk(-(la * c.nxdPt.x + c.dPr.x), -(la * c.nxdPt.y + c.dPr.y), -(la * c.nxdPt.z + c.dPr.z));
    o.Pa = c.Pa;
    o.Pb = c.Pb;
    return o;
}

// The contact-local projected update (half_core, sweep_core.cuh) on stored rows/normals.
__device__ __forceinline__ HalfOut half_contact(const double4 VA, const double4 WA, const double4 VB, const double4 WB,
                                                bool isB, double mt, const G4 g, const R4 rw, const P4 pa,
                                                const P4 pb, int rolling_dims)
{
    return half_core(VA, WA, VB, WB, isB, mt, mk(g.x, g.y, g.z), g.w, rw.x, rw.y, rw.z, rw.w, pa, pb, rolling_dims);
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
