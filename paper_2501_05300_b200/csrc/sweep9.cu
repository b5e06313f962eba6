// sweep9.cu -- staged tile sweep: every contact evaluated once per tile that holds it, all of a
// tile's inputs staged in shared memory by asynchronous copies before any arithmetic.
//
// The measured limiter of the gather sweep (k_sweep_t2) is the L1 data pipe plus the latency of
// dependent gathers: every half-contact re-reads its contact record and both
// bodies' states through per-lane loads.  Here a block owns a tile of T consecutive particles
// (rebuild's level/Morton order) and
//   phase 0  stages, with cp.async (no register round trip, all loads in flight at once):
//            the tile's states; its A-items -- the contacts whose body a is in the tile, one
//            CONTIGUOUS range of the contact arrays (contacts are sorted by a) -- normals, rows,
//            impulses and partner ids; the partner states of A-items whose body b lies outside
//            the tile; its X-items -- the cross-tile contacts whose body b is in the tile (per
//            step lists, k_inc9_*) -- with their records and body-a states;
//   phase 1  evaluates each A-item and each X-item ONCE (one thread per item, one call site of
//            contact_core, so a cross-tile contact evaluated in both of its tiles gives
//            bit-identical impulses); new impulses to shared memory, A-items' to global memory
//            (coalesced: consecutive threads hold consecutive contacts);
//   phase 2  one thread per particle sums its contributions from the impulse increments in a
//            fixed order (its A-items, then its B-halves in incidence order): deterministic, no
//            atomics, no shuffles; the contribution of a contact is rebuilt from (P_new - P_old),
//            the normal and the lever arm exactly as contact_core forms it.
// Intra-tile contacts (about half at T = 64 on the bench bed) are evaluated once instead of twice.
#include "common.cuh"
#include "kernels.h"
#include "sweep_core.cuh"

#ifndef SWEEP9_TILE
#define SWEEP9_TILE 64
#endif
#ifndef SWEEP9_THREADS
#define SWEEP9_THREADS 128
#endif
#ifndef SWEEP9_MINB
#define SWEEP9_MINB 2
#endif
constexpr int T9 = SWEEP9_TILE;
constexpr int NT9 = SWEEP9_THREADS;

// ------------------------------------------------------------------ per-step incidence
// ca[i]: first contact with body a = i; xstart/xlist: cross-tile B-halves per particle
// {contact, body a, 0, local index of body b}; caps[0/1]: largest A / X count of a tile
__global__ void k_inc9_count(int64_t N, const uint32_t *__restrict__ co_start, const uint32_t *__restrict__ cscan,
                             const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                             uint32_t *__restrict__ ca, uint32_t *__restrict__ xcnt)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > N) return;
    const uint32_t a0 = cscan[co_start[i]];
    ca[i] = a0;
    if (i == N) return;
    const uint32_t nb = (inc_start[i + 1] - inc_start[i]) - (cscan[co_start[i + 1]] - a0);
    const uint32_t s = inc_start[i];
    const int64_t ti = i / T9;
    uint32_t x = 0;
    for (uint32_t t = 0; t < nb; t++) x += ((int64_t)inc[s + t].y / T9 != ti) ? 1u : 0u;
    xcnt[i] = x;
}

__global__ void k_inc9_fill(int64_t N, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                            const uint32_t *__restrict__ ca, const uint32_t *__restrict__ xstart,
                            uint4 *__restrict__ xlist)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t nb = (inc_start[i + 1] - inc_start[i]) - (ca[i + 1] - ca[i]), s = inc_start[i];
    const int64_t ti = i / T9;
    uint32_t o = xstart[i];
    for (uint32_t t = 0; t < nb; t++) {
        const uint2 e = inc[s + t];
        if ((int64_t)e.y / T9 != ti) xlist[o++] = make_uint4(e.x & INC_CMASK, e.y, 0u, (uint32_t)(i - ti * T9));
    }
}

__global__ void k_tile_caps9(int64_t N, const uint32_t *__restrict__ ca, const uint32_t *__restrict__ xstart,
                             const uint32_t *__restrict__ inc_start, unsigned int *caps)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t p0 = t * T9;
    if (p0 >= N) return;
    const int64_t p1 = min(p0 + T9, N);
    atomicMax(&caps[0], ca[p1] - ca[p0]);
    atomicMax(&caps[1], xstart[p1] - xstart[p0]);
    atomicMax(&caps[2], inc_start[p1] - inc_start[p0]);
}

// ------------------------------------------------------------------ cp.async helpers
__device__ __forceinline__ void cpa16(void *smem, const void *gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// copy n records of S bytes (S multiple of 16) from g to s, block-strided in 16-byte granules
template <int S>
__device__ __forceinline__ void stage(void *s, const void *g, int n, int t)
{
    constexpr int K = S / 16;
    const int m = n * K;
    for (int q = t; q < m; q += NT9) cpa16((char *)s + 16 * q, (const char *)g + 16 * q);
}

// one record of S bytes by the calling thread
template <int S>
__device__ __forceinline__ void stage1(void *s, const void *g)
{
#pragma unroll
    for (int q = 0; q < S / 16; q++) cpa16((char *)s + 16 * q, (const char *)g + 16 * q);
}

// shared-memory layout (byte offsets from the dynamic base), capacities from the per-step caps
struct Lay9 {
    int capA, capX, capI;
    size_t oInc, oXs, oV, oW, oI, oCa, oAa, oXe, oAg, oAr, oAp, oAq, oAn, oAm, oAb, oAv, oAw, oXg, oXr, oXp, oXq, oXn, oXm, oXv, oXw, total;
    __host__ __device__ Lay9(int a, int x, int ci) : capA(a), capX(x), capI(ci)
    {
        size_t o = 0;
        auto take = [&](size_t bytes) { const size_t r = o; o += (bytes + 15) & ~(size_t)15; return r; };
        oInc = take(sizeof(uint2) * ci);                                 // the tile's incidence entries
        oXs = take(sizeof(uint32_t) * (T9 + 1));                         // X-list starts
        oV = take(sizeof(double4) * T9); oW = take(sizeof(double4) * T9);
        oI = take(sizeof(uint32_t) * (T9 + 1)); oCa = take(sizeof(uint32_t) * (T9 + 1));
        oAa = take(sizeof(uint16_t) * a);                                // body a, tile-local
        oXe = take(sizeof(uint4) * x);
        oAg = take(sizeof(G4) * a); oAr = take(sizeof(R4) * a);
        oAp = take(sizeof(P4) * a); oAq = take(sizeof(P4) * a);          // old P (Pa, Pb)
        oAn = take(sizeof(P4) * a); oAm = take(sizeof(P4) * a);          // new P
        oAb = take(sizeof(uint32_t) * a);                                // partner code
        oAv = take(sizeof(double4) * a); oAw = take(sizeof(double4) * a); // cross partner states
        oXg = take(sizeof(G4) * x); oXr = take(sizeof(R4) * x);
        oXp = take(sizeof(P4) * x); oXq = take(sizeof(P4) * x);
        oXn = take(sizeof(P4) * x); oXm = take(sizeof(P4) * x);
        oXv = take(sizeof(double4) * x); oXw = take(sizeof(double4) * x);
        total = o;
    }
};

template <class T>
__device__ __forceinline__ T *at(unsigned char *b, size_t o) { return reinterpret_cast<T *>(b + o); }

__device__ __forceinline__ d3 pt_of(const P4 p) { return mk(p_ld(p.y), p_ld(p.z), p_ld(p.w)); }
__device__ __forceinline__ d3 pr_of(const P4 p) { return mk(p_ld(p.x), p_ld(p.y), p_ld(p.z)); }

__global__ void __launch_bounds__(NT9, SWEEP9_MINB)
    k_sweep9(int64_t N, int capA, int capX, int capI, const double4 *__restrict__ vin, const double4 *__restrict__ win,
             double4 *__restrict__ vout, double4 *__restrict__ wout, const uint32_t *__restrict__ ca,
             const uint32_t *__restrict__ xstart, const uint4 *__restrict__ xlist, const uint32_t *__restrict__ inc_start,
             const uint2 *__restrict__ inc, const uint2 *__restrict__ cij, const G4 *__restrict__ geo,
             const R4 *__restrict__ row, const P4 *__restrict__ Pa_in, const P4 *__restrict__ Pb_in,
             P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    extern __shared__ __align__(16) unsigned char sm9[];
    const Lay9 L(capA, capX, capI);
    uint2 *sInc = at<uint2>(sm9, L.oInc);
    uint32_t *sXs = at<uint32_t>(sm9, L.oXs);
    double4 *sV = at<double4>(sm9, L.oV), *sW = at<double4>(sm9, L.oW);
    uint32_t *sI = at<uint32_t>(sm9, L.oI), *sCa = at<uint32_t>(sm9, L.oCa), *sAb = at<uint32_t>(sm9, L.oAb);
    uint4 *sXe = at<uint4>(sm9, L.oXe);
    uint16_t *sAa = at<uint16_t>(sm9, L.oAa);
    G4 *sAg = at<G4>(sm9, L.oAg), *sXg = at<G4>(sm9, L.oXg);
    R4 *sAr = at<R4>(sm9, L.oAr), *sXr = at<R4>(sm9, L.oXr);
    P4 *sAp = at<P4>(sm9, L.oAp), *sAq = at<P4>(sm9, L.oAq), *sAn = at<P4>(sm9, L.oAn), *sAm = at<P4>(sm9, L.oAm);
    P4 *sXp = at<P4>(sm9, L.oXp), *sXq = at<P4>(sm9, L.oXq), *sXn = at<P4>(sm9, L.oXn), *sXm = at<P4>(sm9, L.oXm);
    double4 *sAv = at<double4>(sm9, L.oAv), *sAw = at<double4>(sm9, L.oAw);
    double4 *sXv = at<double4>(sm9, L.oXv), *sXw = at<double4>(sm9, L.oXw);

    const int t = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * T9;
    const int np = (int)min((int64_t)T9, N - p0);
    const uint32_t c0 = ca[p0], nA = ca[p0 + np] - c0;
    const uint32_t x0 = xstart[p0], nX = xstart[p0 + np] - x0;

    // ---- phase 0a: contiguous data (tile states, A-item records, X entries), all asynchronous
    stage<32>(sV, vin + p0, np, t);
    stage<32>(sW, win + p0, np, t);
    stage<sizeof(G4)>(sAg, geo + c0, nA, t);
    stage<sizeof(R4)>(sAr, row + c0, nA, t);
    stage<sizeof(P4)>(sAp, Pa_in + c0, nA, t);
    stage<sizeof(P4)>(sAq, Pb_in + c0, nA, t);
    stage<16>(sXe, xlist + x0, nX, t);
    cpa_commit();
    for (int q = t; q <= np; q += NT9) {
        sI[q] = inc_start[p0 + q];
        sCa[q] = ca[p0 + q];
        sXs[q] = xstart[p0 + q] - x0;
    }
    {
        const uint32_t i0 = inc_start[p0], ni = inc_start[p0 + np] - i0;
        for (uint32_t q = t; q < ni; q += NT9) sInc[q] = inc[i0 + q];     // coalesced, read by phase 2
    }
    for (uint32_t q = t; q < nA; q += NT9) {
        const uint2 ij = cij[c0 + q];
        sAb[q] = ij.y;
        sAa[q] = (uint16_t)(ij.x - (uint32_t)p0);
    }
    cpa_wait_all();
    __syncthreads();
    // ---- phase 0b: gathers that need the ids just staged
    for (uint32_t q = t; q < nA; q += NT9) {
        const uint32_t p = sAb[q];
        if (!(p & PARTNER_EXT) && (int64_t)p - p0 >= np) {           // p > a >= p0: cross iff beyond the tile
            stage1<32>(&sAv[q], vin + p);
            stage1<32>(&sAw[q], win + p);
        }
    }
    for (uint32_t k = t; k < nX; k += NT9) {
        const uint4 e = sXe[k];
        stage1<sizeof(G4)>(&sXg[k], geo + e.x);
        stage1<sizeof(R4)>(&sXr[k], row + e.x);
        stage1<sizeof(P4)>(&sXp[k], Pa_in + e.x);
        stage1<sizeof(P4)>(&sXq[k], Pb_in + e.x);
        stage1<32>(&sXv[k], vin + e.y);
        stage1<32>(&sXw[k], win + e.y);
    }
    cpa_commit();
    cpa_wait_all();
    __syncthreads();

    // ---- phase 1: every item evaluated once (single call site of contact_core)
    for (uint32_t q = t; q < nA + nX; q += NT9) {
        const bool isA = q < nA;
        const uint32_t k = q - nA;
        double4 VA, WA, VB, WB;
        uint32_t p;
        G4 g;
        R4 rw;
        P4 pa, pb;
        if (isA) {
            p = sAb[q];
            const int la = sAa[q];
            VA = sV[la]; WA = sW[la];
            if (!(p & PARTNER_EXT)) {
                const int64_t pl = (int64_t)p - p0;
                if (pl < np) { VB = sV[pl]; WB = sW[pl]; }
                else { VB = sAv[q]; WB = sAw[q]; }
            }
            g = sAg[q]; rw = sAr[q]; pa = sAp[q]; pb = sAq[q];
        } else {
            const uint4 e = sXe[k];
            p = 0u;
            VA = sXv[k]; WA = sXw[k];
            VB = sV[e.w]; WB = sW[e.w];
            g = sXg[k]; rw = sXr[k]; pa = sXp[k]; pb = sXq[k];
        }
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
            sAn[q] = r.Pa; sAm[q] = r.Pb;
            Pa_out[c0 + q] = r.Pa;
            Pb_out[c0 + q] = r.Pb;
        } else {
            sXn[k] = r.Pa; sXm[k] = r.Pb;
        }
    }
    __syncthreads();

    // ---- phase 2: per particle, contributions from the impulse increments in a fixed order
    if (t < np) {
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0;
        const uint32_t qa0 = sCa[t] - c0, qa1 = sCa[t + 1] - c0;
        for (uint32_t q = qa0; q < qa1; q++) {            // body a of its A-items
            const G4 g = sAg[q];
            const d3 n = mk(g.x, g.y, g.z);
            const P4 o = sAp[q], nw = sAn[q];
            const double dPn = p_ld(nw.x) - p_ld(o.x);
            const d3 dPt = pt_of(nw) - pt_of(o);
            const d3 dPr = pr_of(sAm[q]) - pr_of(sAq[q]);
            const d3 Lc = dPn * n + dPt;
            const d3 nx = cross(n, dPt);
            const double la = sAr[q].z;
            s0 -= Lc.x; s1 -= Lc.y; s2 -= Lc.z;
            s3 -= la * nx.x + dPr.x; s4 -= la * nx.y + dPr.y; s5 -= la * nx.z + dPr.z;
        }
        // body b of its B-halves (inc lists them first, in partner order)
        const uint32_t nb = (sI[t + 1] - sI[t]) - (qa1 - qa0);
        uint32_t xk = sXs[t];
        const uint32_t ib = sI[t] - sI[0];
        for (uint32_t j = 0; j < nb; j++) {
            const uint2 e = sInc[ib + j];
            const uint32_t c = e.x & INC_CMASK;
            G4 g;
            double lb;
            P4 o, nw, ob, nb2;
            if ((int64_t)e.y - p0 >= 0 && (int64_t)e.y - p0 < np) {
                const uint32_t q = c - c0;
                g = sAg[q]; lb = sAr[q].w; o = sAp[q]; nw = sAn[q]; ob = sAq[q]; nb2 = sAm[q];
            } else {
                g = sXg[xk]; lb = sXr[xk].w; o = sXp[xk]; nw = sXn[xk]; ob = sXq[xk]; nb2 = sXm[xk];
                xk++;
            }
            const d3 n = mk(g.x, g.y, g.z);
            const double dPn = p_ld(nw.x) - p_ld(o.x);
            const d3 dPt = pt_of(nw) - pt_of(o);
            const d3 dPr = pr_of(nb2) - pr_of(ob);
            const d3 Lc = dPn * n + dPt;
            const d3 nx = cross(n, dPt);
            s0 += Lc.x; s1 += Lc.y; s2 += Lc.z;
            s3 += -lb * nx.x + dPr.x; s4 += -lb * nx.y + dPr.y; s5 += -lb * nx.z + dPr.z;
        }
        double4 V = sV[t], W = sW[t];
        const uint32_t cnt = sI[t + 1] - sI[t];
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

// ------------------------------------------------------------------ launchers
void launch_inc9(int64_t N, const uint32_t *co_start, const uint32_t *cscan, const uint32_t *inc_start, const uint2 *inc,
                 uint32_t *ca, uint32_t *xcnt, uint32_t *xstart, uint4 *xlist, unsigned int *caps, void *scan_tmp,
                 cudaStream_t s, long long *launches)
{
    k_inc9_count<<<(unsigned)((N + 1 + 255) / 256), 256, 0, s>>>(N, co_start, cscan, inc_start, inc, ca, xcnt);
    scan_u32(xcnt, xstart, N, scan_tmp, s, launches);
    if (N) k_inc9_fill<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, inc_start, inc, ca, xstart, xlist);
    cudaMemsetAsync(caps, 0, 3 * sizeof(unsigned int), s);
    const int64_t nt = (N + T9 - 1) / T9;
    if (nt) k_tile_caps9<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(N, ca, xstart, inc_start, caps);
    *launches += 3;
}

size_t sweep9_smem_bytes(unsigned capA, unsigned capX, unsigned capI) { return Lay9((int)capA, (int)capX, (int)capI).total; }
int sweep9_tile() { return T9; }

void launch_sweep9(int64_t N, unsigned capA, unsigned capX, unsigned capI, const double4 *vin, const double4 *win, double4 *vout,
                   double4 *wout, const uint32_t *ca, const uint32_t *xstart, const uint4 *xlist,
                   const uint32_t *inc_start, const uint2 *inc, const uint2 *cij, const G4 *geo, const R4 *row,
                   const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out, const DevBoundary *bnd,
                   const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    capA = capA ? capA : 1;
    capX = capX ? capX : 1;
    capI = capI ? capI : 1;
    const size_t smem = sweep9_smem_bytes(capA, capX, capI);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_sweep9, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    k_sweep9<<<(unsigned)((N + T9 - 1) / T9), NT9, smem, s>>>(N, (int)capA, (int)capX, (int)capI, vin, win, vout, wout, ca, xstart,
                                                             xlist, inc_start, inc, cij, geo, row, Pa_in, Pb_in, Pa_out,
                                                             Pb_out, bnd, sp);
}
