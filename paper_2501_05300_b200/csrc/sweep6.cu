// sweep6.cu -- tile-paired Jacobi sweep: every contact whose two bodies lie in the same
// particle tile is evaluated ONCE per sweep.
//
// A block owns a tile of T6 consecutive particles in the (level, Morton) order of the last
// rebuild.  Contacts are stored sorted by body a (the compaction keeps candidate order), so the
// tile's "A-items" -- the contacts whose body a is in the tile -- are one contiguous, coalesced
// range of the contact arrays.  Each A-item is evaluated once:
//   * intra-tile (body b in the tile too): both bodies read from shared memory; body a's
//     contribution enters a's segmented sum, body b's goes to b's shared-memory B-slot;
//   * cross-tile or boundary: the partner is gathered from global memory; only a's
//     contribution is used here (b's tile evaluates the same contact again as a "B-item").
// "B-items" are the cross-tile contacts whose body b is in the tile (per-particle lists built
// once per step, k_inc6_*); their contribution goes to b's B-slot.  A cross-tile contact is
// evaluated from both tiles with identical canonical operands through one call site of
// contact_core, so both ends see bit-identical impulses; body a's tile writes P.
// Each particle finally adds its A-sum (fixed-order segmented shuffle scan, as k_sweep_tile)
// and its B-slots in list order: a deterministic reduction, no float atomics.
// With Morton tiles of 128 particles ~65 % of the bench bed's contacts are intra-tile, so a
// sweep evaluates ~1.35 contacts per contact instead of 2.
#include "common.cuh"
#include "kernels.h"
#include "sweep_core.cuh"

#ifndef SWEEP6_MINB
#define SWEEP6_MINB 3
#endif

// ------------------------------------------------------------------ per-step incidence
// ca[i]     first contact with body a = i (contacts sorted by a): cscan[co_start[i]]
// bstart[i] first B-slot of particle i (B-halves in the order of inc, i.e. by partner a)
//           = inc_start[i] - ca[i] (inc lists a particle's B-halves before its A-halves)
// xcnt[i]   number of i's B-halves whose body a lies in another tile
__global__ void k_inc6_count(int64_t N, int tile, const uint32_t *__restrict__ co_start,
                             const uint32_t *__restrict__ cscan, const uint32_t *__restrict__ inc_start,
                             const uint2 *__restrict__ inc, uint32_t *__restrict__ ca, uint32_t *__restrict__ bstart,
                             uint32_t *__restrict__ xcnt)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > N) return;
    const uint32_t a0 = cscan[co_start[i]];
    ca[i] = a0;
    bstart[i] = inc_start[i] - a0;
    if (i == N) return;
    const uint32_t nb = (inc_start[i + 1] - inc_start[i]) - (cscan[co_start[i + 1]] - a0);
    const uint32_t s = inc_start[i];
    const int64_t ti = i / tile;
    uint32_t x = 0;
    for (uint32_t t = 0; t < nb; t++) x += ((int64_t)inc[s + t].y / tile != ti) ? 1u : 0u;
    xcnt[i] = x;
}

__global__ void k_inc6_fill(int64_t N, int tile, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                            const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ xstart,
                            uint32_t *__restrict__ bslot, uint2 *__restrict__ xlist)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t nb = bstart[i + 1] - bstart[i], s = inc_start[i], b0 = bstart[i];
    const int64_t ti = i / tile;
    uint32_t o = xstart[i];
    for (uint32_t t = 0; t < nb; t++) {
        const uint2 e = inc[s + t];
        const uint32_t c = e.x & INC_CMASK;
        bslot[c] = b0 + t;
        if ((int64_t)e.y / tile != ti) xlist[o++] = make_uint2(c, e.y);
    }
}

// largest B-slot count of a tile (shared-memory size of the sweep launch); integer max
__global__ void k_tile_maxb(int64_t N, int tile, const uint32_t *__restrict__ bstart, unsigned int *out)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t p0 = t * tile;
    if (p0 >= N) return;
    const int64_t p1 = min(p0 + tile, N);
    atomicMax(out, bstart[p1] - bstart[p0]);
}

// ------------------------------------------------------------------ the sweep
// canonical-orientation evaluation of contact (a, b); p = partner code of body b
template <bool IMPACT>
__device__ __forceinline__ ContactOut eval_canon(const double4 XA, const double4 VA, const double4 WA, const double4 XB,
                                                 const double4 VB_, const double4 WB_, uint32_t p, double b,
                                                 const P4 pa, const P4 pb, const DevBoundary *__restrict__ bnd,
                                                 const SolveParams &sp, double &la, double &lb)
{
    d3 n;
    double delta, mt, mr, Rs;
    double4 VB = VB_, WB = WB_;
    if (!(p & PARTNER_EXT)) {
        pair_geom(XA, XB, n, delta);
        Rs = rstar(XA.w, XB.w);
        la = XA.w - 0.5 * delta;
        lb = XB.w - 0.5 * delta;
        mt = sp.mu_t;
        mr = sp.mu_r;
    } else {
        ext_geom(XA, p & ~PARTNER_EXT, bnd, n, delta);
        d3 bv;
        boundary_body(p, bnd, bv, mt, mr);
        Rs = XA.w;
        la = XA.w - 0.5 * delta;
        lb = 0.0;
        VB = make_double4(bv.x, bv.y, bv.z, 0.0);
        WB = make_double4(0.0, 0.0, 0.0, 0.0);
    }
    const double S = IMPACT ? 0.0 : spook_sigma(sp, Rs, delta);
    return contact_core(VA, WA, VB, WB, mt, n, mr * Rs, S, b, la, lb, pa, pb, sp.rolling_dims);
}

template <int TILE>
struct Smem6 {
    static constexpr int NW = TILE / 32;
    double4 sX[TILE], sV[TILE], sW[TILE];
    double sAcc[NW][6][32];
    uint32_t sCa[TILE + 1], sXs[TILE + 1], sBs[TILE + 1];
    uint8_t sOwnA[NW][32], sOwnX[NW][32];
};

template <int TILE>
size_t sweep6_smem(unsigned max_b) { return sizeof(Smem6<TILE>) + (size_t)6 * max_b * sizeof(double); }

template <int TILE, bool IMPACT>
__global__ void __launch_bounds__(TILE, TILE == 256 ? 2 : SWEEP6_MINB)
    k_sweep6(int64_t N, int cap, const double4 *__restrict__ pos, const double4 *__restrict__ vin,
             const double4 *__restrict__ win, double4 *__restrict__ vout, double4 *__restrict__ wout,
             const uint32_t *__restrict__ ca, const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ xstart,
             const uint2 *__restrict__ xlist, const uint2 *__restrict__ cij, const uint32_t *__restrict__ bslot,
             const double *__restrict__ cb, const P4 *__restrict__ Pa_in, const P4 *__restrict__ Pb_in,
             P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    extern __shared__ __align__(16) unsigned char smraw[];
    Smem6<TILE> &sm = *reinterpret_cast<Smem6<TILE> *>(smraw);
    double *slot = reinterpret_cast<double *>(smraw + sizeof(Smem6<TILE>));   // [6][cap]
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * TILE;
    const int np = (int)min((int64_t)TILE, N - p0);
    if (t < np) {
        sm.sX[t] = pos[p0 + t];
        sm.sV[t] = vin[p0 + t];
        sm.sW[t] = win[p0 + t];
    }
    for (int q = t; q <= np; q += TILE) {
        sm.sCa[q] = ca[p0 + q];
        sm.sXs[q] = xstart[p0 + q];
        sm.sBs[q] = bstart[p0 + q];
    }
#pragma unroll
    for (int f = 0; f < 6; f++) sm.sAcc[w][f][lane] = 0.0;
    __syncthreads();
    const uint32_t base = sm.sBs[0];
    const int lo_p = 32 * w, hi_p = min(32 * w + 32, np);
    const int me = lo_p + lane;
    const bool mine = me < hi_p;
    if (lo_p < np) {
        const uint32_t a0 = sm.sCa[lo_p], a1 = sm.sCa[hi_p], x0 = sm.sXs[lo_p], x1 = sm.sXs[hi_p];
        const uint32_t nA = a1 - a0, nT = nA + (x1 - x0);
        // this lane's particle: A-range and cross-B range, in the warp's item numbering
        const uint32_t aS = mine ? sm.sCa[me] - a0 : 0u, aE = mine ? sm.sCa[me + 1] - a0 : 0u;
        const uint32_t xS = mine ? nA + sm.sXs[me] - x0 : 0u, xE = mine ? nA + sm.sXs[me + 1] - x0 : 0u;
        int carryA = 0, carryX = 0;
        for (uint32_t kb = 0; kb < nT; kb += 32) {
            const uint32_t k = kb + lane;
            const bool valid = k < nT, isA = k < nA;
            const bool stA = aE > aS && aS >= kb && aS < kb + 32;
            const bool stX = xE > xS && xS >= kb && xS < kb + 32;
            const unsigned mA = __reduce_or_sync(0xffffffffu, stA ? (1u << (aS - kb)) : 0u);
            const unsigned mX = __reduce_or_sync(0xffffffffu, stX ? (1u << (xS - kb)) : 0u);
            if (stA) sm.sOwnA[w][aS - kb] = (uint8_t)lane;
            if (stX) sm.sOwnX[w][xS - kb] = (uint8_t)lane;
            __syncwarp();
            const unsigned upto = 0xffffffffu >> (31 - lane);
            const unsigned leA = mA & upto, leX = mX & upto;
            const int sA = leA ? 31 - __clz(leA) : 0;
            const int ownerA = leA ? (int)sm.sOwnA[w][sA] : carryA;
            const int ownerX = leX ? (int)sm.sOwnX[w][31 - __clz(leX)] : carryX;
            double v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, v5 = 0;
            if (valid) {
                uint32_t c, p;
                int oself;
                double4 XA, VA, WA, XB, VB, WB;
                bool intra = false;
                if (isA) {
                    c = a0 + k;
                    p = cij[c].y;
                    oself = lo_p + ownerA;
                    XA = sm.sX[oself]; VA = sm.sV[oself]; WA = sm.sW[oself];
                    if (!(p & PARTNER_EXT)) {
                        const int64_t pl = (int64_t)p - p0;
                        intra = pl >= 0 && pl < np;
                        if (intra) { XB = sm.sX[pl]; VB = sm.sV[pl]; WB = sm.sW[pl]; }
                        else { XB = pos[p]; VB = vin[p]; WB = win[p]; }
                    }
                } else {
                    const uint2 e = xlist[x0 + (k - nA)];
                    c = e.x;
                    p = 0u;                       // body b is this tile's particle
                    oself = lo_p + ownerX;
                    XA = pos[e.y]; VA = vin[e.y]; WA = win[e.y];
                    XB = sm.sX[oself]; VB = sm.sV[oself]; WB = sm.sW[oself];
                }
                double la, lb;
                const ContactOut r = eval_canon<IMPACT>(XA, VA, WA, XB, VB, WB, p, cb[c], Pa_in[c], Pb_in[c], bnd, sp, la, lb);
                if (isA) {
                    Pa_out[c] = r.Pa;
                    Pb_out[c] = r.Pb;
                    v0 = -r.L.x; v1 = -r.L.y; v2 = -r.L.z;
                    v3 = -(la * r.nxdPt.x + r.dPr.x); v4 = -(la * r.nxdPt.y + r.dPr.y); v5 = -(la * r.nxdPt.z + r.dPr.z);
                }
                if (!isA || intra) {
                    const uint32_t q = bslot[c] - base;
                    slot[0 * cap + q] = r.L.x;
                    slot[1 * cap + q] = r.L.y;
                    slot[2 * cap + q] = r.L.z;
                    slot[3 * cap + q] = -lb * r.nxdPt.x + r.dPr.x;
                    slot[4 * cap + q] = -lb * r.nxdPt.y + r.dPr.y;
                    slot[5 * cap + q] = -lb * r.nxdPt.z + r.dPr.z;
                }
            }
            // segmented inclusive scan of the A-items, depth = longest A segment of the chunk
            const int dist = (valid && isA) ? lane - sA : 0;
            const int maxd = __reduce_max_sync(0xffffffffu, dist);
            for (int d = 1; d <= maxd; d <<= 1) {
                const double u0 = __shfl_up_sync(0xffffffffu, v0, d), u1 = __shfl_up_sync(0xffffffffu, v1, d);
                const double u2 = __shfl_up_sync(0xffffffffu, v2, d), u3 = __shfl_up_sync(0xffffffffu, v3, d);
                const double u4 = __shfl_up_sync(0xffffffffu, v4, d), u5 = __shfl_up_sync(0xffffffffu, v5, d);
                if (lane - d >= sA) { v0 += u0; v1 += u1; v2 += u2; v3 += u3; v4 += u4; v5 += u5; }
            }
            const bool seg_end = valid && isA && (lane == 31 || ((mA >> (lane + 1)) & 1u) || k + 1 >= nA);
            if (seg_end) {
                sm.sAcc[w][0][ownerA] += v0; sm.sAcc[w][1][ownerA] += v1; sm.sAcc[w][2][ownerA] += v2;
                sm.sAcc[w][3][ownerA] += v3; sm.sAcc[w][4][ownerA] += v4; sm.sAcc[w][5][ownerA] += v5;
            }
            carryA = __shfl_sync(0xffffffffu, ownerA, 31);
            carryX = __shfl_sync(0xffffffffu, ownerX, 31);
            __syncwarp();
        }
    }
    __syncthreads();
    if (t < np) {
        // A-sum, then the B-slots in list order (by partner): fixed order -> bit-reproducible
        double s0 = sm.sAcc[w][0][lane], s1 = sm.sAcc[w][1][lane], s2 = sm.sAcc[w][2][lane];
        double s3 = sm.sAcc[w][3][lane], s4 = sm.sAcc[w][4][lane], s5 = sm.sAcc[w][5][lane];
        const uint32_t q0 = sm.sBs[t] - base, q1 = sm.sBs[t + 1] - base;
        for (uint32_t q = q0; q < q1; q++) {
            s0 += slot[0 * cap + q]; s1 += slot[1 * cap + q]; s2 += slot[2 * cap + q];
            s3 += slot[3 * cap + q]; s4 += slot[4 * cap + q]; s5 += slot[5 * cap + q];
        }
        double4 V = sm.sV[t], W = sm.sW[t];
        const uint32_t cnt = (sm.sCa[t + 1] - sm.sCa[t]) + (q1 - q0);
        if (cnt) {
            // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            V.x += im * s0; V.y += im * s1; V.z += im * s2;
            W.x += iI * s3; W.y += iI * s4; W.z += iI * s5;
        }
        vout[p0 + t] = V;
        wout[p0 + t] = W;
    }
}


#ifndef SWEEP7_MINB
#define SWEEP7_MINB 4
#endif
template <int TILE>
__global__ void __launch_bounds__(TILE, SWEEP7_MINB)
    k_sweep7(int64_t N, int cap, const double4 *__restrict__ pos, const double4 *__restrict__ vin,
             const double4 *__restrict__ win, double4 *__restrict__ vout, double4 *__restrict__ wout,
             const uint32_t *__restrict__ ca, const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ xstart,
             const uint2 *__restrict__ xlist, const uint2 *__restrict__ cij, const uint32_t *__restrict__ bslot,
             const G4 *__restrict__ geo, const R4 *__restrict__ row, const P4 *__restrict__ Pa_in, const P4 *__restrict__ Pb_in,
             P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    extern __shared__ __align__(16) unsigned char smraw[];
    Smem6<TILE> &sm = *reinterpret_cast<Smem6<TILE> *>(smraw);
    double *slot = reinterpret_cast<double *>(smraw + sizeof(Smem6<TILE>));   // [6][cap]
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * TILE;
    const int np = (int)min((int64_t)TILE, N - p0);
    if (t < np) {
        sm.sV[t] = ld4g(&vin[p0 + t]);
        sm.sW[t] = ld4g(&win[p0 + t]);
    }
    for (int q = t; q <= np; q += TILE) {
        sm.sCa[q] = ca[p0 + q];
        sm.sXs[q] = xstart[p0 + q];
        sm.sBs[q] = bstart[p0 + q];
    }
#pragma unroll
    for (int f = 0; f < 6; f++) sm.sAcc[w][f][lane] = 0.0;
    __syncthreads();
    const uint32_t base = sm.sBs[0];
    const int lo_p = 32 * w, hi_p = min(32 * w + 32, np);
    const int me = lo_p + lane;
    const bool mine = me < hi_p;
    if (lo_p < np) {
        const uint32_t a0 = sm.sCa[lo_p], a1 = sm.sCa[hi_p], x0 = sm.sXs[lo_p], x1 = sm.sXs[hi_p];
        const uint32_t nA = a1 - a0, nT = nA + (x1 - x0);
        // this lane's particle: A-range and cross-B range, in the warp's item numbering
        const uint32_t aS = mine ? sm.sCa[me] - a0 : 0u, aE = mine ? sm.sCa[me + 1] - a0 : 0u;
        const uint32_t xS = mine ? nA + sm.sXs[me] - x0 : 0u, xE = mine ? nA + sm.sXs[me + 1] - x0 : 0u;
        int carryA = 0, carryX = 0;
        for (uint32_t kb = 0; kb < nT; kb += 32) {
            const uint32_t k = kb + lane;
            const bool valid = k < nT, isA = k < nA;
            const bool stA = aE > aS && aS >= kb && aS < kb + 32;
            const bool stX = xE > xS && xS >= kb && xS < kb + 32;
            const unsigned mA = __reduce_or_sync(0xffffffffu, stA ? (1u << (aS - kb)) : 0u);
            const unsigned mX = __reduce_or_sync(0xffffffffu, stX ? (1u << (xS - kb)) : 0u);
            if (stA) sm.sOwnA[w][aS - kb] = (uint8_t)lane;
            if (stX) sm.sOwnX[w][xS - kb] = (uint8_t)lane;
            __syncwarp();
            const unsigned upto = 0xffffffffu >> (31 - lane);
            const unsigned leA = mA & upto, leX = mX & upto;
            const int sA = leA ? 31 - __clz(leA) : 0;
            const int ownerA = leA ? (int)sm.sOwnA[w][sA] : carryA;
            const int ownerX = leX ? (int)sm.sOwnX[w][31 - __clz(leX)] : carryX;
            double v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, v5 = 0;
            if (valid) {
                uint32_t c, p;
                int oself;
                double4 VA, WA, VB, WB;
                bool intra = false;
                if (isA) {
                    c = a0 + k;
                    p = cij[c].y;
                    oself = lo_p + ownerA;
                    VA = sm.sV[oself]; WA = sm.sW[oself];
                    if (!(p & PARTNER_EXT)) {
                        const int64_t pl = (int64_t)p - p0;
                        intra = pl >= 0 && pl < np;
                        if (intra) { VB = sm.sV[pl]; WB = sm.sW[pl]; }
                        else { VB = ld4g(&vin[p]); WB = ld4g(&win[p]); }
                    }
                } else {
                    const uint2 e = xlist[x0 + (k - nA)];
                    c = e.x;
                    p = 0u;                       // body b is this tile's particle
                    oself = lo_p + ownerX;
                    VA = ld4g(&vin[e.y]); WA = ld4g(&win[e.y]);
                    VB = sm.sV[oself]; WB = sm.sW[oself];
                }
                const G4 g = ld4g(&geo[c]);
                const R4 rw = ld4g(&row[c]);
                double mt = sp.mu_t;
                if (p & PARTNER_EXT) {
                    d3 bv;
                    double mr;
                    boundary_body(p, bnd, bv, mt, mr);
                    VB = make_double4(bv.x, bv.y, bv.z, 0.0);
                    WB = make_double4(0.0, 0.0, 0.0, 0.0);
                }
                const double la = rw.z, lb = rw.w;
                const ContactOut r = contact_core(VA, WA, VB, WB, mt, mk(g.x, g.y, g.z), g.w, rw.x, rw.y, la, lb,
                                                  Pa_in[c], Pb_in[c], sp.rolling_dims);
                if (isA) {
                    Pa_out[c] = r.Pa;
                    Pb_out[c] = r.Pb;
                    v0 = -r.L.x; v1 = -r.L.y; v2 = -r.L.z;
                    v3 = -(la * r.nxdPt.x + r.dPr.x); v4 = -(la * r.nxdPt.y + r.dPr.y); v5 = -(la * r.nxdPt.z + r.dPr.z);
                }
                if (!isA || intra) {
                    const uint32_t q = bslot[c] - base;
                    slot[0 * cap + q] = r.L.x;
                    slot[1 * cap + q] = r.L.y;
                    slot[2 * cap + q] = r.L.z;
                    slot[3 * cap + q] = -lb * r.nxdPt.x + r.dPr.x;
                    slot[4 * cap + q] = -lb * r.nxdPt.y + r.dPr.y;
                    slot[5 * cap + q] = -lb * r.nxdPt.z + r.dPr.z;
                }
            }
            // segmented inclusive scan of the A-items, depth = longest A segment of the chunk
            const int dist = (valid && isA) ? lane - sA : 0;
            const int maxd = __reduce_max_sync(0xffffffffu, dist);
            for (int d = 1; d <= maxd; d <<= 1) {
                const double u0 = __shfl_up_sync(0xffffffffu, v0, d), u1 = __shfl_up_sync(0xffffffffu, v1, d);
                const double u2 = __shfl_up_sync(0xffffffffu, v2, d), u3 = __shfl_up_sync(0xffffffffu, v3, d);
                const double u4 = __shfl_up_sync(0xffffffffu, v4, d), u5 = __shfl_up_sync(0xffffffffu, v5, d);
                if (lane - d >= sA) { v0 += u0; v1 += u1; v2 += u2; v3 += u3; v4 += u4; v5 += u5; }
            }
            const bool seg_end = valid && isA && (lane == 31 || ((mA >> (lane + 1)) & 1u) || k + 1 >= nA);
            if (seg_end) {
                sm.sAcc[w][0][ownerA] += v0; sm.sAcc[w][1][ownerA] += v1; sm.sAcc[w][2][ownerA] += v2;
                sm.sAcc[w][3][ownerA] += v3; sm.sAcc[w][4][ownerA] += v4; sm.sAcc[w][5][ownerA] += v5;
            }
            carryA = __shfl_sync(0xffffffffu, ownerA, 31);
            carryX = __shfl_sync(0xffffffffu, ownerX, 31);
            __syncwarp();
        }
    }
    __syncthreads();
    if (t < np) {
        // A-sum, then the B-slots in list order (by partner): fixed order -> bit-reproducible
        double s0 = sm.sAcc[w][0][lane], s1 = sm.sAcc[w][1][lane], s2 = sm.sAcc[w][2][lane];
        double s3 = sm.sAcc[w][3][lane], s4 = sm.sAcc[w][4][lane], s5 = sm.sAcc[w][5][lane];
        const uint32_t q0 = sm.sBs[t] - base, q1 = sm.sBs[t + 1] - base;
        for (uint32_t q = q0; q < q1; q++) {
            s0 += slot[0 * cap + q]; s1 += slot[1 * cap + q]; s2 += slot[2 * cap + q];
            s3 += slot[3 * cap + q]; s4 += slot[4 * cap + q]; s5 += slot[5 * cap + q];
        }
        double4 V = sm.sV[t], W = sm.sW[t];
        const uint32_t cnt = (sm.sCa[t + 1] - sm.sCa[t]) + (q1 - q0);
        if (cnt) {
            // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            V.x += im * s0; V.y += im * s1; V.z += im * s2;
            W.x += iI * s3; W.y += iI * s4; W.z += iI * s5;
        }
        st4g(&vout[p0 + t], V);
        st4g(&wout[p0 + t], W);
    }
}


void launch_sweep7(int64_t N, unsigned max_b, const double4 *vin, const double4 *win, double4 *vout, double4 *wout,
                   const uint32_t *ca, const uint32_t *bstart, const uint32_t *xstart, const uint2 *xlist,
                   const uint2 *cij, const uint32_t *bslot, const G4 *geo, const R4 *row, const P4 *Pa_in,
                   const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out, const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    if (max_b == 0) max_b = 1;
    const size_t smem = sweep6_smem<128>(max_b);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_sweep7<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    k_sweep7<128><<<(unsigned)((N + 127) / 128), 128, smem, s>>>(N, (int)max_b, nullptr, vin, win, vout, wout, ca, bstart,
                                                               xstart, xlist, cij, bslot, geo, row, Pa_in, Pb_in, Pa_out,
                                                               Pb_out, bnd, sp);
}
// ------------------------------------------------------------------ launchers
void launch_inc6(int64_t N, int tile, const uint32_t *co_start, const uint32_t *cscan, const uint32_t *inc_start,
                 const uint2 *inc, uint32_t *ca, uint32_t *bstart, uint32_t *xcnt, uint32_t *xstart, uint32_t *bslot,
                 uint2 *xlist, unsigned int *max_b, void *scan_tmp, cudaStream_t s, long long *launches)
{
    k_inc6_count<<<(unsigned)((N + 1 + 255) / 256), 256, 0, s>>>(N, tile, co_start, cscan, inc_start, inc, ca, bstart, xcnt);
    scan_u32(xcnt, xstart, N, scan_tmp, s, launches);
    if (N) k_inc6_fill<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, tile, inc_start, inc, bstart, xstart, bslot, xlist);
    cudaMemsetAsync(max_b, 0, sizeof(unsigned int), s);
    const int64_t nt = (N + tile - 1) / tile;
    if (nt) k_tile_maxb<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(N, tile, bstart, max_b);
    *launches += 3;
}

size_t sweep6_smem_bytes(int tile, unsigned max_b)
{
    return tile == 256 ? sweep6_smem<256>(max_b) : sweep6_smem<128>(max_b);
}

template <int TILE, bool IMPACT>
static void launch6(int64_t N, unsigned max_b, const double4 *pos, const double4 *vin, const double4 *win, double4 *vout,
                    double4 *wout, const uint32_t *ca, const uint32_t *bstart, const uint32_t *xstart,
                    const uint2 *xlist, const uint2 *cij, const uint32_t *bslot, const double *cb, const P4 *Pa_in,
                    const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out, const DevBoundary *bnd, const SolveParams &sp,
                    cudaStream_t s)
{
    const size_t smem = sweep6_smem<TILE>(max_b);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_sweep6<TILE, IMPACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    k_sweep6<TILE, IMPACT><<<(unsigned)((N + TILE - 1) / TILE), TILE, smem, s>>>(
        N, (int)max_b, pos, vin, win, vout, wout, ca, bstart, xstart, xlist, cij, bslot, cb, Pa_in, Pb_in, Pa_out, Pb_out,
        bnd, sp);
}

void launch_sweep6(int tile, bool impact, int64_t N, unsigned max_b, const double4 *pos, const double4 *vin,
                   const double4 *win, double4 *vout, double4 *wout, const uint32_t *ca, const uint32_t *bstart,
                   const uint32_t *xstart, const uint2 *xlist, const uint2 *cij, const uint32_t *bslot,
                   const double *cb, const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out,
                   const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    if (max_b == 0) max_b = 1;
#define A6 N, max_b, pos, vin, win, vout, wout, ca, bstart, xstart, xlist, cij, bslot, cb, Pa_in, Pb_in, Pa_out, Pb_out, bnd, sp, s
    if (tile == 256) {
        if (impact) launch6<256, true>(A6); else launch6<256, false>(A6);
    } else {
        if (impact) launch6<128, true>(A6); else launch6<128, false>(A6);
    }
#undef A6
}

// ==================================================================== slot sweep (v8)
// Same tile pairing as k_sweep6, but the tile's items are spread over ALL threads of the block
// (block-strided loop; A-items are consecutive contacts -> coalesced loads) and every
// contribution goes to a shared-memory slot: A-slot q for the q-th A-item of the tile, B-slot
// for the B-half.  No segmented scan and no owner search: after one barrier each particle sums
// its A-slots and then its B-slots in list order (fixed order -> bit-reproducible).  Normals
// and row constants are read from the stored contact arrays (streamed for A-items).
struct XItem { uint32_t c, a, bslot, pad; };

__global__ void k_inc8_fill(int64_t N, int tile, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                            const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ xstart,
                            uint32_t *__restrict__ bslot, uint4 *__restrict__ xlist)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t nb = bstart[i + 1] - bstart[i], s = inc_start[i], b0 = bstart[i];
    const int64_t ti = i / tile;
    uint32_t o = xstart[i];
    for (uint32_t t = 0; t < nb; t++) {
        const uint2 e = inc[s + t];
        const uint32_t c = e.x & INC_CMASK;
        bslot[c] = b0 + t;
        if ((int64_t)e.y / tile != ti) xlist[o++] = make_uint4(c, e.y, b0 + t, (uint32_t)(i - ti * tile));
    }
}

// largest A + B slot count of a tile
__global__ void k_tile_maxslots(int64_t N, int tile, const uint32_t *__restrict__ ca, const uint32_t *__restrict__ bstart,
                                unsigned int *out)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t p0 = t * tile;
    if (p0 >= N) return;
    const int64_t p1 = min(p0 + tile, N);
    atomicMax(out, (ca[p1] - ca[p0]) + (bstart[p1] - bstart[p0]));
}

#ifndef SWEEP8_TILE
#define SWEEP8_TILE 128
#endif
#ifndef SWEEP8_MINB
#define SWEEP8_MINB 3
#endif
constexpr int T8 = SWEEP8_TILE;

struct Smem8 {
    double4 sV[T8], sW[T8];
    uint32_t sCa[T8 + 1], sBs[T8 + 1];
};

__global__ void __launch_bounds__(T8, SWEEP8_MINB)
    k_sweep8(int64_t N, int cap, const double4 *__restrict__ vin, const double4 *__restrict__ win,
             double4 *__restrict__ vout, double4 *__restrict__ wout, const uint32_t *__restrict__ ca,
             const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ xstart, const uint4 *__restrict__ xlist,
             const uint2 *__restrict__ cij, const uint32_t *__restrict__ bslot, const G4 *__restrict__ geo,
             const R4 *__restrict__ row, const P4 *__restrict__ Pa_in, const P4 *__restrict__ Pb_in,
             P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    extern __shared__ __align__(16) unsigned char smraw[];
    Smem8 &sm = *reinterpret_cast<Smem8 *>(smraw);
    double *slot = reinterpret_cast<double *>(smraw + sizeof(Smem8));   // [6][cap]: A-slots, then B-slots
    const int t = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * T8;
    const int np = (int)min((int64_t)T8, N - p0);
    if (t < np) {
        sm.sV[t] = vin[p0 + t];
        sm.sW[t] = win[p0 + t];
    }
    for (int q = t; q <= np; q += T8) {
        sm.sCa[q] = ca[p0 + q];
        sm.sBs[q] = bstart[p0 + q];
    }
    const uint32_t x0 = xstart[p0], x1 = xstart[p0 + np];
    __syncthreads();
    const uint32_t c0 = sm.sCa[0], nA = sm.sCa[np] - c0, base = sm.sBs[0];
    const uint32_t nT = nA + (x1 - x0);
    // item descriptors one iteration ahead: {contact, partner, B-slot, self (tile-local)}
    auto fetch = [&](uint32_t q) -> uint4 {
        if (q < nA) {
            const uint32_t c = c0 + q;
            const uint2 ij = cij[c];
            return make_uint4(c, ij.y, bslot[c], ij.x - (uint32_t)p0);
        }
        return xlist[x0 + (q - nA)];
    };
    uint4 dnext = t < nT ? fetch(t) : make_uint4(0, 0, 0, 0);
    for (uint32_t q = t; q < nT; q += T8) {
        const bool isA = q < nA;
        const uint4 d = dnext;
        if (q + T8 < nT) dnext = fetch(q + T8);
        const uint32_t c = d.x, sb = d.z;
        const int self = (int)d.w;
        uint32_t p;
        bool intra = false;
        double4 VA, WA, VB, WB;
        if (isA) {
            p = d.y;
            VA = sm.sV[self]; WA = sm.sW[self];
            if (!(p & PARTNER_EXT)) {
                const int64_t pl = (int64_t)p - p0;
                intra = pl < np;                     // p > a >= p0
                if (intra) { VB = sm.sV[pl]; WB = sm.sW[pl]; }
                else { VB = vin[p]; WB = win[p]; }
            }
        } else {
            p = 0u;
            VA = vin[d.y]; WA = win[d.y];
            VB = sm.sV[self]; WB = sm.sW[self];
        }
        const G4 g = geo[c];
        const R4 rw = row[c];
        const P4 pa = Pa_in[c], pb = Pb_in[c];
        double mt = sp.mu_t;
        if (p & PARTNER_EXT) {
            d3 bv;
            double mr;
            boundary_body(p, bnd, bv, mt, mr);
            VB = make_double4(bv.x, bv.y, bv.z, 0.0);
            WB = make_double4(0.0, 0.0, 0.0, 0.0);
        }
        const ContactOut r = contact_core(VA, WA, VB, WB, mt, mk(g.x, g.y, g.z), g.w, rw.x, rw.y, rw.z, rw.w, pa, pb,
                                          sp.rolling_dims);
        if (isA) {
            Pa_out[c] = r.Pa;
            Pb_out[c] = r.Pb;
            const double la = rw.z;
            slot[0 * cap + q] = -r.L.x;
            slot[1 * cap + q] = -r.L.y;
            slot[2 * cap + q] = -r.L.z;
            slot[3 * cap + q] = -(la * r.nxdPt.x + r.dPr.x);
            slot[4 * cap + q] = -(la * r.nxdPt.y + r.dPr.y);
            slot[5 * cap + q] = -(la * r.nxdPt.z + r.dPr.z);
        }
        if (!isA || intra) {
            const uint32_t s = nA + (sb - base);
            const double lb = rw.w;
            slot[0 * cap + s] = r.L.x;
            slot[1 * cap + s] = r.L.y;
            slot[2 * cap + s] = r.L.z;
            slot[3 * cap + s] = -lb * r.nxdPt.x + r.dPr.x;
            slot[4 * cap + s] = -lb * r.nxdPt.y + r.dPr.y;
            slot[5 * cap + s] = -lb * r.nxdPt.z + r.dPr.z;
        }
    }
    __syncthreads();
    if (t < np) {
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0;
        const uint32_t qa0 = sm.sCa[t] - c0, qa1 = sm.sCa[t + 1] - c0;
        const uint32_t qb0 = nA + sm.sBs[t] - base, qb1 = nA + sm.sBs[t + 1] - base;
        for (uint32_t q = qa0; q < qa1; q++) {
            s0 += slot[0 * cap + q]; s1 += slot[1 * cap + q]; s2 += slot[2 * cap + q];
            s3 += slot[3 * cap + q]; s4 += slot[4 * cap + q]; s5 += slot[5 * cap + q];
        }
        for (uint32_t q = qb0; q < qb1; q++) {
            s0 += slot[0 * cap + q]; s1 += slot[1 * cap + q]; s2 += slot[2 * cap + q];
            s3 += slot[3 * cap + q]; s4 += slot[4 * cap + q]; s5 += slot[5 * cap + q];
        }
        double4 V = sm.sV[t], W = sm.sW[t];
        const uint32_t cnt = (qa1 - qa0) + (qb1 - qb0);
        if (cnt) {
            // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            V.x += im * s0; V.y += im * s1; V.z += im * s2;
            W.x += iI * s3; W.y += iI * s4; W.z += iI * s5;
        }
        vout[p0 + t] = V;
        wout[p0 + t] = W;
    }
}

void launch_inc8(int64_t N, const uint32_t *co_start, const uint32_t *cscan, const uint32_t *inc_start, const uint2 *inc,
                 uint32_t *ca, uint32_t *bstart, uint32_t *xcnt, uint32_t *xstart, uint32_t *bslot, uint4 *xlist,
                 unsigned int *max_slots, void *scan_tmp, cudaStream_t s, long long *launches)
{
    k_inc6_count<<<(unsigned)((N + 1 + 255) / 256), 256, 0, s>>>(N, T8, co_start, cscan, inc_start, inc, ca, bstart, xcnt);
    scan_u32(xcnt, xstart, N, scan_tmp, s, launches);
    if (N) k_inc8_fill<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, T8, inc_start, inc, bstart, xstart, bslot, xlist);
    cudaMemsetAsync(max_slots, 0, sizeof(unsigned int), s);
    const int64_t nt = (N + T8 - 1) / T8;
    if (nt) k_tile_maxslots<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(N, T8, ca, bstart, max_slots);
    *launches += 3;
}

size_t sweep8_smem_bytes(unsigned max_slots) { return sizeof(Smem8) + (size_t)6 * max_slots * sizeof(double); }

void launch_sweep8(int64_t N, unsigned max_slots, const double4 *vin, const double4 *win, double4 *vout, double4 *wout,
                   const uint32_t *ca, const uint32_t *bstart, const uint32_t *xstart, const uint4 *xlist,
                   const uint2 *cij, const uint32_t *bslot, const G4 *geo, const R4 *row, const P4 *Pa_in,
                   const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out, const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    if (max_slots == 0) max_slots = 1;
    const size_t smem = sweep8_smem_bytes(max_slots);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_sweep8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    k_sweep8<<<(unsigned)((N + T8 - 1) / T8), T8, smem, s>>>(N, (int)max_slots, vin, win, vout, wout, ca, bstart, xstart,
                                                               xlist, cij, bslot, geo, row, Pa_in, Pb_in, Pa_out, Pb_out,
                                                               bnd, sp);
}
