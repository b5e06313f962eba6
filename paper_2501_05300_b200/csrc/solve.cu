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

// ------------------------------------------------------------------ the Jacobi sweep

constexpr int TP = 128;
constexpr int NW = TP / 32;
#ifndef SWEEP_MINB
#define SWEEP_MINB 5
#endif
#ifndef SWEEP_MINB_PIPE
#define SWEEP_MINB_PIPE 3
#endif
#ifndef SWEEP_MINB_PPT
#define SWEEP_MINB_PPT 4
#endif
#ifndef SWEEP_KERNEL
#define SWEEP_KERNEL 0      // 0: k_sweep_t2 (default, fastest measured), 1: k_sweep_pipe, 2: k_sweep_ppt, 4: k_sweep_tile
#endif

// Tile sweep: the block stages the tile's states and CSR offsets in shared memory once; each
// warp then owns 32 consecutive particles and walks their half-contacts 32 at a time, with no
// block barrier inside the loop.  Per chunk, owners come from a warp-wide bitmask of segment
// starts; the lanes' contributions are reduced per owner by a segmented shuffle scan whose
// depth is the longest segment of the chunk, and each segment's last lane adds the sum to the
// owner's warp-private shared accumulator (one writer per particle per chunk): a fixed
// summation order, hence deterministic, and no float atomics.
__device__ __forceinline__ void pf_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// EXP (timing experiments only): 1 no contact math, 2 no contact-record loads, 3 neither
// contact-record nor partner global loads (math on shared memory only)
__device__ __forceinline__ HalfOut fake_half(const double4 VA, const double4 WA, const double4 VB, const double4 WB,
                                             const G4 g, const R4 rw, const P4 pa, const P4 pb)
{
    HalfOut o;
    o.dL = mk(1e-30 * (VA.x + VB.x + g.x + rw.x + pa.x), 1e-30 * (VA.y + WB.y + g.y + rw.y + pb.x),
              1e-30 * (WA.z + VB.z + g.z + rw.z + pa.y));
    o.dA = mk(1e-30 * (WA.x + g.w + rw.w + pa.z), 1e-30 * (WB.x + pa.w + pb.y), 1e-30 * pb.z);
    o.Pa = pa;
    o.Pb = pb;
    return o;
}

template <bool PF, int EXP = 0>
__global__ void __launch_bounds__(TP, SWEEP_MINB) k_sweep_tile(int64_t N, const double4 *__restrict__ vin,
                                                      const double4 *__restrict__ win, double4 *__restrict__ vout,
                                                      double4 *__restrict__ wout, const uint32_t *__restrict__ inc_start,
                                                      const uint2 *__restrict__ inc, const G4 *__restrict__ geo,
                                                      const R4 *__restrict__ row, const P4 *__restrict__ Pa_in,
                                                      const P4 *__restrict__ Pb_in, P4 *__restrict__ Pa_out,
                                                      P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd,
                                                      SolveParams sp)
{
    __shared__ double4 sV[TP], sW[TP];
    __shared__ double4 sExt[TP];                     // per lane: boundary-body velocity
    __shared__ double sAcc[NW][6][32];               // per warp: per-particle accumulators
    __shared__ uint8_t sOwn[NW][32];                 // per warp: owner of each segment start
    __shared__ uint32_t sI[TP + 1];
    __shared__ double4 sZero;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * TP;
    const int np = (int)min((int64_t)TP, N - p0);
    if (t < np) {
        sV[t] = vin[p0 + t];
        sW[t] = win[p0 + t];
    }
    for (int q = t; q <= np; q += TP) sI[q] = inc_start[p0 + q];
    if (t == 0) sZero = make_double4(0, 0, 0, 0);
#pragma unroll
    for (int f = 0; f < 6; f++) sAcc[w][f][lane] = 0.0;
    __syncthreads();
    const int lo_p = 32 * w, hi_p = min(32 * w + 32, np);
    const int me = lo_p + lane;                      // this lane's particle (if me < hi_p)
    const uint32_t s_me = me < hi_p ? sI[me] : 0u, e_me = me < hi_p ? sI[me + 1] : 0u;
    if (lo_p < np) {
        const uint32_t k0 = sI[lo_p], k1 = sI[hi_p];
        uint2 ent_next = make_uint2(0, 0), ent_nn = make_uint2(0, 0);
        if (k0 + lane < k1) ent_next = inc[k0 + lane];
        if (PF && k0 + 32 + lane < k1) ent_nn = inc[k0 + 32 + lane];
        int carry = 0;                               // owner (warp-local) of the chunk's lane 0
        for (uint32_t kb = k0; kb < k1; kb += 32) {
            const uint32_t k = kb + lane;
            const bool valid = k < k1;
            const uint2 ent = ent_next;
            if (PF) {
                // L1 prefetch of the next chunk's contact records and partner states while this
                // chunk computes; incidence two chunks ahead in registers
                ent_next = ent_nn;
                if (kb + 32 + lane < k1) {
                    const uint32_t c2 = ent_next.x & INC_CMASK, p2 = ent_next.y;
                    pf_l1(&geo[c2]); pf_l1(&row[c2]); pf_l1(&Pa_in[c2]); pf_l1(&Pb_in[c2]);
                    if (!(p2 & PARTNER_EXT)) {
                        const int64_t pl = (int64_t)p2 - p0;
                        if (pl < 0 || pl >= np) { pf_l1(&vin[p2]); pf_l1(&win[p2]); }
                    }
                }
                if (kb + 64 + lane < k1) ent_nn = inc[kb + 64 + lane];
            } else if (kb + 32 + lane < k1) ent_next = inc[kb + 32 + lane];     // prefetch the next chunk
            // segment starts of this chunk (nonempty particles whose CSR range starts here)
            const bool starts = e_me > s_me && s_me >= kb && s_me < kb + 32;
            const unsigned smask = __reduce_or_sync(0xffffffffu, starts ? (1u << (s_me - kb)) : 0u);
            if (starts) sOwn[w][s_me - kb] = (uint8_t)lane;
            __syncwarp();
            const unsigned le = smask & (0xffffffffu >> (31 - lane));
            const int sstart = le ? 31 - __clz(le) : 0;
            const int owner = le ? (int)sOwn[w][sstart] : carry;
            double v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, v5 = 0;
            if (valid) {
                const int o = lo_p + owner;
                const uint32_t c = ent.x & INC_CMASK;
                const bool isB = (ent.x & B_SIDE) != 0;
                const uint32_t p = ent.y;
                const double4 *pPV, *pPW;
                double mt;
                if (!(p & PARTNER_EXT)) {
                    const int64_t pl = EXP == 3 ? (int64_t)(p & (TP - 1)) : (int64_t)p - p0;
                    if (pl >= 0 && pl < np) { pPV = &sV[pl]; pPW = &sW[pl]; }
                    else { pPV = &vin[p]; pPW = &win[p]; }
                    mt = sp.mu_t;
                } else {
                    d3 bv;
                    boundary_vel(p, bnd, bv, mt);
                    sExt[t] = make_double4(bv.x, bv.y, bv.z, 0.0);
                    pPV = &sExt[t];
                    pPW = &sZero;
                }
                const double4 *pSV = &sV[o], *pSW = &sW[o];
                G4 gc;
                R4 rc;
                P4 pac, pbc;
                if (EXP >= 2) {
                    gc = mkG4(0.6, 0.0, 0.8, 1e-4 + 1e-12 * c);
                    rc = mkR4(1e5, 1e-3, 1e-3, 1e-3);
                    pac = mkP4(1e-6, 0, 0, 0);
                    pbc = mkP4(0, 0, 0, 0);
                } else {
                    gc = geo[c]; rc = row[c]; pac = Pa_in[c]; pbc = Pb_in[c];
                }
                const HalfOut r = EXP == 1 ? fake_half(*(isB ? pPV : pSV), *(isB ? pPW : pSW), *(isB ? pSV : pPV),
                                                       *(isB ? pSW : pPW), gc, rc, pac, pbc)
                                           : half_contact(*(isB ? pPV : pSV), *(isB ? pPW : pSW), *(isB ? pSV : pPV),
                                               *(isB ? pSW : pPW), isB, mt, gc, rc, pac, pbc,
                                               sp.rolling_dims);
                if (!isB) {
                    Pa_out[c] = r.Pa;
                    Pb_out[c] = r.Pb;
                }
                v0 = r.dL.x; v1 = r.dL.y; v2 = r.dL.z; v3 = r.dA.x; v4 = r.dA.y; v5 = r.dA.z;
            }
            // segmented inclusive scan, depth = longest segment of this chunk
            const int dist = valid ? lane - sstart : 0;
            const int maxd = __reduce_max_sync(0xffffffffu, dist);
            for (int d = 1; d <= maxd; d <<= 1) {
                const double u0 = __shfl_up_sync(0xffffffffu, v0, d), u1 = __shfl_up_sync(0xffffffffu, v1, d);
                const double u2 = __shfl_up_sync(0xffffffffu, v2, d), u3 = __shfl_up_sync(0xffffffffu, v3, d);
                const double u4 = __shfl_up_sync(0xffffffffu, v4, d), u5 = __shfl_up_sync(0xffffffffu, v5, d);
                if (lane - d >= sstart) { v0 += u0; v1 += u1; v2 += u2; v3 += u3; v4 += u4; v5 += u5; }
            }
            const bool seg_end = valid && (lane == 31 || ((smask >> (lane + 1)) & 1u) || k + 1 >= k1);
            if (seg_end) {
                sAcc[w][0][owner] += v0; sAcc[w][1][owner] += v1; sAcc[w][2][owner] += v2;
                sAcc[w][3][owner] += v3; sAcc[w][4][owner] += v4; sAcc[w][5][owner] += v5;
            }
            carry = __shfl_sync(0xffffffffu, owner, 31);
            __syncwarp();
        }
    }
    if (me < hi_p) {
        // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
        double4 V = sV[me], W = sW[me];
        const uint32_t cnt = e_me - s_me;
        if (cnt) {
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            V.x += im * sAcc[w][0][lane]; V.y += im * sAcc[w][1][lane]; V.z += im * sAcc[w][2][lane];
            W.x += iI * sAcc[w][3][lane]; W.y += iI * sAcc[w][4][lane]; W.z += iI * sAcc[w][5][lane];
        }
        vout[p0 + me] = V;
        wout[p0 + me] = W;
    }
}

// ------------------------------------------------------------------ pipelined tile sweep
// Same work split and reduction as k_sweep_tile, plus a 2-stage cp.async pipeline: while a
// warp computes chunk i it has chunk i+1's contact records (geo, row, P) and partner states in
// flight into a warp-private shared-memory stage (LDGSTS, L2-only), and chunk i+2's incidence
// entries in registers.  Load latency is then hidden by the warp's own computation instead of
// by occupancy.
__device__ __forceinline__ void cp16(void *smem, const void *gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
template <class T>
__device__ __forceinline__ void cpT(T *smem, const T *gmem)
{
    static_assert(sizeof(T) % 16 == 0, "16-byte granules");
#pragma unroll
    for (int q = 0; q < (int)(sizeof(T) / 16); q++) cp16((char *)smem + 16 * q, (const char *)gmem + 16 * q);
}

struct Stage {                      // one chunk of one warp (SoA: conflict-free per-lane access)
    G4 geo[32];
    R4 row[32];
    P4 pa[32], pb[32];
    double4 vp[32], wp[32];
};
constexpr int TPP = 128;
constexpr int NWP = TPP / 32;
struct PipeSmem {
    Stage st[NWP][2];
    double4 sV[TPP], sW[TPP];
    double sAcc[NWP][6][32];
    uint32_t sI[TPP + 1];
    uint8_t sOwn[NWP][32];
};
size_t sweep_pipe_smem() { return sizeof(PipeSmem); }

__device__ __forceinline__ void issue_stage(Stage &S, int lane, bool valid, uint2 ent, const G4 *__restrict__ geo,
                                            const R4 *__restrict__ row, const P4 *__restrict__ Pa,
                                            const P4 *__restrict__ Pb, const double4 *__restrict__ vin,
                                            const double4 *__restrict__ win)
{
    if (!valid) return;
    const uint32_t c = ent.x & INC_CMASK, p = ent.y;
    cpT(&S.geo[lane], &geo[c]);
    cpT(&S.row[lane], &row[c]);
    cpT(&S.pa[lane], &Pa[c]);
    cpT(&S.pb[lane], &Pb[c]);
    if (!(p & PARTNER_EXT)) {
        cpT(&S.vp[lane], &vin[p]);
        cpT(&S.wp[lane], &win[p]);
    }
}

__global__ void __launch_bounds__(TPP, SWEEP_MINB_PIPE) k_sweep_pipe(int64_t N, const double4 *__restrict__ vin,
                                                      const double4 *__restrict__ win, double4 *__restrict__ vout,
                                                      double4 *__restrict__ wout, const uint32_t *__restrict__ inc_start,
                                                      const uint2 *__restrict__ inc, const G4 *__restrict__ geo,
                                                      const R4 *__restrict__ row, const P4 *__restrict__ Pa_in,
                                                      const P4 *__restrict__ Pb_in, P4 *__restrict__ Pa_out,
                                                      P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd,
                                                      SolveParams sp)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PipeSmem &sm = *reinterpret_cast<PipeSmem *>(smem_raw);
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * TPP;
    const int np = (int)min((int64_t)TPP, N - p0);
    if (t < np) {
        sm.sV[t] = vin[p0 + t];
        sm.sW[t] = win[p0 + t];
    }
    for (int q = t; q <= np; q += TPP) sm.sI[q] = inc_start[p0 + q];
#pragma unroll
    for (int f = 0; f < 6; f++) sm.sAcc[w][f][lane] = 0.0;
    __syncthreads();
    const int lo_p = 32 * w, hi_p = min(32 * w + 32, np);
    const int me = lo_p + lane;
    const uint32_t s_me = me < hi_p ? sm.sI[me] : 0u, e_me = me < hi_p ? sm.sI[me + 1] : 0u;
    if (lo_p < np) {
        const uint32_t k0 = sm.sI[lo_p], k1 = sm.sI[hi_p];
        uint2 entA = make_uint2(0, 0), entB = make_uint2(0, 0);
        if (k0 + lane < k1) entA = inc[k0 + lane];
        if (k0 + 32 + lane < k1) entB = inc[k0 + 32 + lane];
        issue_stage(sm.st[w][0], lane, k0 + lane < k1, entA, geo, row, Pa_in, Pb_in, vin, win);
        cp_commit();
        int carry = 0;
        int sidx = 0;
        for (uint32_t kb = k0; kb < k1; kb += 32) {
            const uint32_t k = kb + lane;
            const bool valid = k < k1;
            // stage chunk i+1, prefetch the incidence of chunk i+2
            issue_stage(sm.st[w][sidx ^ 1], lane, kb + 32 + lane < k1, entB, geo, row, Pa_in, Pb_in, vin, win);
            cp_commit();
            uint2 entC = make_uint2(0, 0);
            if (kb + 64 + lane < k1) entC = inc[kb + 64 + lane];
            // owners of this chunk's lanes from the segment-start bitmask
            const bool starts = e_me > s_me && s_me >= kb && s_me < kb + 32;
            const unsigned smask = __reduce_or_sync(0xffffffffu, starts ? (1u << (s_me - kb)) : 0u);
            if (starts) sm.sOwn[w][s_me - kb] = (uint8_t)lane;
            cp_wait1();
            __syncwarp();
            const unsigned le = smask & (0xffffffffu >> (31 - lane));
            const int sstart = le ? 31 - __clz(le) : 0;
            const int owner = le ? (int)sm.sOwn[w][sstart] : carry;
            double v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, v5 = 0;
            if (valid) {
                Stage &S = sm.st[w][sidx];
                const int o = lo_p + owner;
                const bool isB = (entA.x & B_SIDE) != 0;
                const uint32_t p = entA.y;
                double mt;
                double4 VP, WP;
                if (!(p & PARTNER_EXT)) {
                    VP = S.vp[lane];
                    WP = S.wp[lane];
                    mt = sp.mu_t;
                } else {
                    d3 bv;
                    boundary_vel(p, bnd, bv, mt);
                    VP = make_double4(bv.x, bv.y, bv.z, 0.0);
                    WP = make_double4(0.0, 0.0, 0.0, 0.0);
                }
                const double4 VS = sm.sV[o], WS = sm.sW[o];
                const HalfOut r = half_contact(isB ? VP : VS, isB ? WP : WS, isB ? VS : VP, isB ? WS : WP, isB, mt,
                                               S.geo[lane], S.row[lane], S.pa[lane], S.pb[lane], sp.rolling_dims);
                if (!isB) {
                    const uint32_t c = entA.x & INC_CMASK;
                    Pa_out[c] = r.Pa;
                    Pb_out[c] = r.Pb;
                }
                v0 = r.dL.x; v1 = r.dL.y; v2 = r.dL.z; v3 = r.dA.x; v4 = r.dA.y; v5 = r.dA.z;
            }
            const int dist = valid ? lane - sstart : 0;
            const int maxd = __reduce_max_sync(0xffffffffu, dist);
            for (int d = 1; d <= maxd; d <<= 1) {
                const double u0 = __shfl_up_sync(0xffffffffu, v0, d), u1 = __shfl_up_sync(0xffffffffu, v1, d);
                const double u2 = __shfl_up_sync(0xffffffffu, v2, d), u3 = __shfl_up_sync(0xffffffffu, v3, d);
                const double u4 = __shfl_up_sync(0xffffffffu, v4, d), u5 = __shfl_up_sync(0xffffffffu, v5, d);
                if (lane - d >= sstart) { v0 += u0; v1 += u1; v2 += u2; v3 += u3; v4 += u4; v5 += u5; }
            }
            const bool seg_end = valid && (lane == 31 || ((smask >> (lane + 1)) & 1u) || k + 1 >= k1);
            if (seg_end) {
                sm.sAcc[w][0][owner] += v0; sm.sAcc[w][1][owner] += v1; sm.sAcc[w][2][owner] += v2;
                sm.sAcc[w][3][owner] += v3; sm.sAcc[w][4][owner] += v4; sm.sAcc[w][5][owner] += v5;
            }
            carry = __shfl_sync(0xffffffffu, owner, 31);
            entA = entB;
            entB = entC;
            sidx ^= 1;
            __syncwarp();
        }
    }
    if (me < hi_p) {
        double4 V = sm.sV[me], W = sm.sW[me];
        const uint32_t cnt = e_me - s_me;
        if (cnt) {
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            V.x += im * sm.sAcc[w][0][lane]; V.y += im * sm.sAcc[w][1][lane]; V.z += im * sm.sAcc[w][2][lane];
            W.x += iI * sm.sAcc[w][3][lane]; W.y += iI * sm.sAcc[w][4][lane]; W.z += iI * sm.sAcc[w][5][lane];
        }
        vout[p0 + me] = V;
        wout[p0 + me] = W;
    }
}

// ------------------------------------------------------------------ particle-per-thread sweep
// One thread per particle walks its own CSR list: contributions accumulate in registers in CSR
// order (deterministic, no reduction step, no owner search).  Divergence from unequal contact
// counts is removed by k_tile_order, which sorts the particles of every 128-tile by count once
// per step, so a warp's lanes have (nearly) equal trip counts.
constexpr int TPT = 128;

__global__ void k_tile_order(int64_t N, const uint32_t *__restrict__ inc_start, uint32_t *__restrict__ order)
{
    __shared__ uint32_t key[TPT];
    const int t = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * TPT;
    const int np = (int)min((int64_t)TPT, N - p0);
    // key = (count << 8) | local index, descending count; padding sorts last
    key[t] = t < np ? (((inc_start[p0 + t + 1] - inc_start[p0 + t]) << 8) | (uint32_t)t) : 0u;
    __syncthreads();
    for (int k = 2; k <= TPT; k <<= 1)           // bitonic sort, descending
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int ix = t ^ j;
            if (ix > t) {
                const uint32_t a = key[t], b = key[ix];
                const bool desc = (t & k) == 0;
                if (desc ? (a < b) : (a > b)) { key[t] = b; key[ix] = a; }
            }
            __syncthreads();
        }
    if (t < np) order[p0 + t] = (uint32_t)(p0 + (key[t] & 0xFF));
}

__global__ void __launch_bounds__(TPT, SWEEP_MINB_PPT) k_sweep_ppt(int64_t N, const uint32_t *__restrict__ order,
                                                      const double4 *__restrict__ vin, const double4 *__restrict__ win,
                                                      double4 *__restrict__ vout, double4 *__restrict__ wout,
                                                      const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                                                      const G4 *__restrict__ geo, const R4 *__restrict__ row,
                                                      const P4 *__restrict__ Pa_in, const P4 *__restrict__ Pb_in,
                                                      P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out,
                                                      const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    const int64_t tid = (int64_t)blockIdx.x * TPT + threadIdx.x;
    if (tid >= N) return;
    const uint32_t i = order[tid];
    const uint32_t s = inc_start[i], e = inc_start[i + 1];
    const double4 V = vin[i], W = win[i];
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
    uint2 ent_next = s < e ? inc[s] : make_uint2(0, 0);
    for (uint32_t k = s; k < e; k++) {
        const uint2 ent = ent_next;
        if (k + 1 < e) ent_next = inc[k + 1];
        const uint32_t c = ent.x & INC_CMASK;
        const bool isB = (ent.x & B_SIDE) != 0;
        const uint32_t p = ent.y;
        double4 VP, WP;
        double mt;
        if (!(p & PARTNER_EXT)) {
            VP = vin[p];
            WP = win[p];
            mt = sp.mu_t;
        } else {
            d3 bv;
            boundary_vel(p, bnd, bv, mt);
            VP = make_double4(bv.x, bv.y, bv.z, 0.0);
            WP = make_double4(0.0, 0.0, 0.0, 0.0);
        }
        const HalfOut r = half_contact(isB ? VP : V, isB ? WP : W, isB ? V : VP, isB ? W : WP, isB, mt, geo[c], row[c],
                                       Pa_in[c], Pb_in[c], sp.rolling_dims);
        if (!isB) {
            Pa_out[c] = r.Pa;
            Pb_out[c] = r.Pb;
        }
        a0 += r.dL.x; a1 += r.dL.y; a2 += r.dL.z; a3 += r.dA.x; a4 += r.dA.y; a5 += r.dA.z;
    }
    double4 Vn = V, Wn = W;
    const uint32_t cnt = e - s;
    if (cnt) {
        const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
        Vn.x += im * a0; Vn.y += im * a1; Vn.z += im * a2;
        Wn.x += iI * a3; Wn.y += iI * a4; Wn.z += iI * a5;
    }
    vout[i] = Vn;
    wout[i] = Wn;
}

static thread_local int g_sweep_variant = SWEEP_KERNEL;   // per host thread: contexts may step concurrently
void set_sweep_variant(int v) { g_sweep_variant = v; }
bool sweep_uses_order() { return g_sweep_variant == 2; }
void launch_tile_order(int64_t N, const uint32_t *inc_start, uint32_t *order, cudaStream_t s)
{ if (N) k_tile_order<<<(unsigned)((N + TPT - 1) / TPT), TPT, 0, s>>>(N, inc_start, order); }

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
template <bool P8L>
__global__ void k_plate_hub(int64_t n, const uint32_t *__restrict__ list, const uint2 *__restrict__ cij,
                            const G4 *__restrict__ geo, const void *__restrict__ pin, const void *__restrict__ pout,
                            unsigned long long *__restrict__ acc)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t c = list[t];
    const int q = (cij[c].y >> 4) & 0xF;
    const G4 g = geo[c];
    const P4 o = P8L ? ((const P8 *)pout)[c].a : ((const P4 *)pout)[c];
    P4 i = mkP4(0, 0, 0, 0);
    if (pin) i = P8L ? ((const P8 *)pin)[c].a : ((const P4 *)pin)[c];
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
void launch_plate_hub(bool p8, int64_t n, const uint32_t *list, const uint2 *cij, const G4 *geo, const void *pin,
                      const void *pout, unsigned long long *acc, cudaStream_t s)
{
    if (!n) return;
    if (p8) k_plate_hub<true><<<PGRID(n)>>>(n, list, cij, geo, pin, pout, acc);
    else k_plate_hub<false><<<PGRID(n)>>>(n, list, cij, geo, pin, pout, acc);
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
void launch_sweep(int mode, int64_t N, const uint32_t *order, const double4 *vin, const double4 *win, double4 *vout,
                  double4 *wout, const uint32_t *inc_start, const uint2 *inc, const PackedInc *pk, const G4 *geo,
                  const R4 *row,
                  const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out,
                  const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    if (mode == SWEEP_MODE_SWEEP && g_sweep_variant == 2) {
        k_sweep_ppt<<<(unsigned)((N + TPT - 1) / TPT), TPT, 0, s>>>(N, order, vin, win, vout, wout, inc_start, inc, geo,
                                                                    row, Pa_in, Pb_in, Pa_out, Pb_out, bnd, sp);
    } else if (mode == SWEEP_MODE_SWEEP && g_sweep_variant == 1) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_sweep_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PipeSmem));
            attr = true;
        }
        k_sweep_pipe<<<(unsigned)((N + TPP - 1) / TPP), TPP, sizeof(PipeSmem), s>>>(
            N, vin, win, vout, wout, inc_start, inc, geo, row, Pa_in, Pb_in, Pa_out, Pb_out, bnd, sp);
    } else if (mode == SWEEP_MODE_SWEEP && (g_sweep_variant == 0 || g_sweep_variant == 7 || g_sweep_variant == 8 ||
                                            g_sweep_variant == 9 || g_sweep_variant == 44 || g_sweep_variant == 45)) {
        // 0: the context's reduction (packed canonical if pk, else contiguous); 7: contiguous;
        // 8: packed with contact-indexed normals/rows (diagnostic; pk->geo/row set by the caller)
        g_t2_rows_by_contact = g_sweep_variant == 8;
        g_t2_stage = g_sweep_variant == 9;
        g_t2_exp = g_sweep_variant == 44 ? 1 : (g_sweep_variant == 45 ? 2 : 0);
        launch_sweep_t2(N, vin, win, vout, wout, inc_start, inc, g_sweep_variant == 7 ? nullptr : pk, geo, row, Pa_in,
                        Pb_in, Pa_out, Pb_out, bnd, sp, s);
        g_t2_rows_by_contact = false;
        g_t2_stage = false;
        g_t2_exp = 0;
    }
    else if (mode == SWEEP_MODE_SWEEP)
        (g_sweep_variant == 3 ? k_sweep_tile<true> : g_sweep_variant == 41 ? k_sweep_tile<false, 1> :
         g_sweep_variant == 42 ? k_sweep_tile<false, 2> : g_sweep_variant == 43 ? k_sweep_tile<false, 3> : k_sweep_tile<false>)<<<(unsigned)((N + TP - 1) / TP), TP, 0, s>>>(N, vin, win, vout, wout, inc_start, inc, geo, row,
                                                                  Pa_in, Pb_in, Pa_out, Pb_out, bnd, sp);
    else if (mode == SWEEP_MODE_APPLY)
        k_apply<SWEEP_MODE_APPLY><<<GRID(N)>>>(N, vin, win, vout, wout, inc_start, inc, geo, row, Pa_in, Pb_in, sp);
    else
        k_apply<SWEEP_MODE_FORCES><<<GRID(N)>>>(N, vin, win, vout, wout, inc_start, inc, geo, row, Pa_in, Pb_in, sp);
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
