// sweep5.cu -- Jacobi sweep kernels that re-evaluate the contact geometry from the particle
// positions instead of streaming stored normals and row constants.
//
// Per sweep a contact needs its unit normal n, overlap delta, lever arms, R* and the SPOOK
// regularisation Sigma-hat; all of them are functions of the two (fixed during the step's
// sweeps) positions and radii, evaluated with the narrow phase's own instruction sequence
// (pair_geom / ext_geom, common.cuh) so they are bit-identical to the stored values.  Only the
// step-dependent bias b (it holds u_n at the step start, reading R4) and the impulses P are
// per-contact data: 8 + 32 B read + 32 B written per contact instead of 64 + 32 + 32 B, at the
// price of one more 32 B position gather per half-contact (an L1/L2 hit for a Morton-local
// partner) and ~40 fp64 operations.
//
//  k_sweep5_ppt   one thread per particle walks its CSR list (tile-local count ordering keeps
//                 the warp's trip counts equal); contributions summed in registers in CSR order
//                 (deterministic, no reduction step); optional 2-stage register prefetch
//  k_sweep5_tile  warp-chunked half-contacts with the segmented shuffle reduction of
//                 k_sweep_tile, tile positions/velocities staged in shared memory
#include "common.cuh"
#include "kernels.h"
#include "sweep_core.cuh"

// One half-contact from the self particle's side.  XS/VS/WS: self, XP/VP/WP: partner particle
// (ignored for a wall/plate partner p).  Canonical orientation a = cij.x, b = cij.y.
template <bool IMPACT>
__device__ __forceinline__ HalfOut eval5(const double4 XS, const double4 VS, const double4 WS, const double4 XP,
                                         const double4 VP, const double4 WP, bool isB, uint32_t p, double b,
                                         const P4 pa, const P4 pb, const DevBoundary *__restrict__ bnd,
                                         const SolveParams &sp)
{
    d3 n;
    double delta, mt, mr, Rs, la, lb;
    double4 VA, WA, VB, WB;
    if (!(p & PARTNER_EXT)) {
        const double4 XA = isB ? XP : XS, XB = isB ? XS : XP;
        pair_geom(XA, XB, n, delta);
        Rs = rstar(XA.w, XB.w);
        la = XA.w - 0.5 * delta;
        lb = XB.w - 0.5 * delta;
        mt = sp.mu_t;
        mr = sp.mu_r;
        VA = isB ? VP : VS; WA = isB ? WP : WS;
        VB = isB ? VS : VP; WB = isB ? WS : WP;
    } else {
        // boundary partner: self is body a; the boundary has zero weights (infinite mass)
        ext_geom(XS, p & ~PARTNER_EXT, bnd, n, delta);
        d3 bv;
        boundary_body(p, bnd, bv, mt, mr);
        Rs = XS.w;
        la = XS.w - 0.5 * delta;
        lb = 0.0;
        VA = VS; WA = WS;
        VB = make_double4(bv.x, bv.y, bv.z, 0.0);
        WB = make_double4(0.0, 0.0, 0.0, 0.0);
    }
    const double S = IMPACT ? 0.0 : spook_sigma(sp, Rs, delta);
    return half_core(VA, WA, VB, WB, isB, mt, n, mr * Rs, S, b, la, lb, pa, pb, sp.rolling_dims);
}

#ifndef SWEEP5_MINB
#define SWEEP5_MINB 4
#endif
constexpr int T5 = 128;

struct Ld5 {
    double4 XP, VP, WP;
    double b;
    P4 pa, pb;
};

__device__ __forceinline__ void ld5(Ld5 &L, uint2 ent, const double4 *__restrict__ pos, const double4 *__restrict__ vin,
                                    const double4 *__restrict__ win, const double *__restrict__ cb,
                                    const P4 *__restrict__ Pa, const P4 *__restrict__ Pb)
{
    const uint32_t c = ent.x & INC_CMASK, p = ent.y;
    L.b = cb[c];
    L.pa = Pa[c];
    L.pb = Pb[c];
    if (!(p & PARTNER_EXT)) {
        L.XP = pos[p];
        L.VP = vin[p];
        L.WP = win[p];
    }
}

template <bool IMPACT, bool PF>
__global__ void __launch_bounds__(T5, PF ? 3 : SWEEP5_MINB)
    k_sweep5_ppt(int64_t N, const uint32_t *__restrict__ order, const double4 *__restrict__ pos,
                 const double4 *__restrict__ vin, const double4 *__restrict__ win, double4 *__restrict__ vout,
                 double4 *__restrict__ wout, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                 const double *__restrict__ cb, const P4 *__restrict__ Pa_in, const P4 *__restrict__ Pb_in,
                 P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    const int64_t tid = (int64_t)blockIdx.x * T5 + threadIdx.x;
    if (tid >= N) return;
    const uint32_t i = order[tid];
    const uint32_t s = inc_start[i], e = inc_start[i + 1];
    const double4 X = pos[i], V = vin[i], W = win[i];
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
    if (PF) {
        Ld5 cur, nxt;
        uint2 ent = s < e ? inc[s] : make_uint2(0, 0);
        uint2 ent_n = s + 1 < e ? inc[s + 1] : make_uint2(0, 0);
        if (s < e) ld5(cur, ent, pos, vin, win, cb, Pa_in, Pb_in);
        for (uint32_t k = s; k < e; k++) {
            uint2 ent_nn = make_uint2(0, 0);
            if (k + 1 < e) ld5(nxt, ent_n, pos, vin, win, cb, Pa_in, Pb_in);
            if (k + 2 < e) ent_nn = inc[k + 2];
            const uint32_t c = ent.x & INC_CMASK;
            const bool isB = (ent.x & B_SIDE) != 0;
            const HalfOut r = eval5<IMPACT>(X, V, W, cur.XP, cur.VP, cur.WP, isB, ent.y, cur.b, cur.pa, cur.pb, bnd, sp);
            if (!isB) {
                Pa_out[c] = r.Pa;
                Pb_out[c] = r.Pb;
            }
            a0 += r.dL.x; a1 += r.dL.y; a2 += r.dL.z; a3 += r.dA.x; a4 += r.dA.y; a5 += r.dA.z;
            cur = nxt;
            ent = ent_n;
            ent_n = ent_nn;
        }
    } else {
        for (uint32_t k = s; k < e; k++) {
            const uint2 ent = inc[k];
            Ld5 L;
            ld5(L, ent, pos, vin, win, cb, Pa_in, Pb_in);
            const uint32_t c = ent.x & INC_CMASK;
            const bool isB = (ent.x & B_SIDE) != 0;
            const HalfOut r = eval5<IMPACT>(X, V, W, L.XP, L.VP, L.WP, isB, ent.y, L.b, L.pa, L.pb, bnd, sp);
            if (!isB) {
                Pa_out[c] = r.Pa;
                Pb_out[c] = r.Pb;
            }
            a0 += r.dL.x; a1 += r.dL.y; a2 += r.dL.z; a3 += r.dA.x; a4 += r.dA.y; a5 += r.dA.z;
        }
    }
    double4 Vn = V, Wn = W;
    const uint32_t cnt = e - s;
    if (cnt) {
        // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
        const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
        Vn.x += im * a0; Vn.y += im * a1; Vn.z += im * a2;
        Wn.x += iI * a3; Wn.y += iI * a4; Wn.z += iI * a5;
    }
    vout[i] = Vn;
    wout[i] = Wn;
}

// warp-chunked variant (the work split and deterministic segmented reduction of k_sweep_tile)
#ifndef SWEEP5T_MINB
#define SWEEP5T_MINB 4
#endif
constexpr int NW5 = T5 / 32;

template <bool IMPACT>
__global__ void __launch_bounds__(T5, SWEEP5T_MINB)
    k_sweep5_tile(int64_t N, const double4 *__restrict__ pos, const double4 *__restrict__ vin,
                  const double4 *__restrict__ win, double4 *__restrict__ vout, double4 *__restrict__ wout,
                  const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc, const double *__restrict__ cb,
                  const P4 *__restrict__ Pa_in, const P4 *__restrict__ Pb_in, P4 *__restrict__ Pa_out,
                  P4 *__restrict__ Pb_out, const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    __shared__ double4 sX[T5], sV[T5], sW[T5];
    __shared__ double sAcc[NW5][6][32];
    __shared__ uint8_t sOwn[NW5][32];
    __shared__ uint32_t sI[T5 + 1];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * T5;
    const int np = (int)min((int64_t)T5, N - p0);
    if (t < np) {
        sX[t] = pos[p0 + t];
        sV[t] = vin[p0 + t];
        sW[t] = win[p0 + t];
    }
    for (int q = t; q <= np; q += T5) sI[q] = inc_start[p0 + q];
#pragma unroll
    for (int f = 0; f < 6; f++) sAcc[w][f][lane] = 0.0;
    __syncthreads();
    const int lo_p = 32 * w, hi_p = min(32 * w + 32, np);
    const int me = lo_p + lane;
    const uint32_t s_me = me < hi_p ? sI[me] : 0u, e_me = me < hi_p ? sI[me + 1] : 0u;
    if (lo_p < np) {
        const uint32_t k0 = sI[lo_p], k1 = sI[hi_p];
        uint2 ent_next = make_uint2(0, 0);
        if (k0 + lane < k1) ent_next = inc[k0 + lane];
        int carry = 0;
        for (uint32_t kb = k0; kb < k1; kb += 32) {
            const uint32_t k = kb + lane;
            const bool valid = k < k1;
            const uint2 ent = ent_next;
            if (kb + 32 + lane < k1) ent_next = inc[kb + 32 + lane];
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
                double4 XP, VP, WP;
                if (!(p & PARTNER_EXT)) {
                    const int64_t pl = (int64_t)p - p0;
                    if (pl >= 0 && pl < np) { XP = sX[pl]; VP = sV[pl]; WP = sW[pl]; }
                    else { XP = pos[p]; VP = vin[p]; WP = win[p]; }
                }
                const HalfOut r = eval5<IMPACT>(sX[o], sV[o], sW[o], XP, VP, WP, isB, p, cb[c], Pa_in[c], Pb_in[c], bnd, sp);
                if (!isB) {
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
                sAcc[w][0][owner] += v0; sAcc[w][1][owner] += v1; sAcc[w][2][owner] += v2;
                sAcc[w][3][owner] += v3; sAcc[w][4][owner] += v4; sAcc[w][5][owner] += v5;
            }
            carry = __shfl_sync(0xffffffffu, owner, 31);
            __syncwarp();
        }
    }
    if (me < hi_p) {
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

// bias column of the row arrays (main rows R4.y) -> cb (bench / migration helper)
__global__ void k_row_bias(int64_t nc, const R4 *__restrict__ row, double *__restrict__ cb)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nc) cb[c] = row[c].y;
}

// max |a.xyz - b.xyz| and max |b.xyz| (non-negative doubles order like their bit patterns)
__global__ void k_maxdiff(int64_t N, const double4 *__restrict__ a, const double4 *__restrict__ b,
                          unsigned long long *out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double d = 0, m = 0;
    if (i < N) {
        const double4 x = a[i], y = b[i];
        d = fmax(fabs(x.x - y.x), fmax(fabs(x.y - y.y), fabs(x.z - y.z)));
        m = fmax(fabs(y.x), fmax(fabs(y.y), fabs(y.z)));
    }
    for (int o = 16; o > 0; o >>= 1) {
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out[0], (unsigned long long)__double_as_longlong(d));
        atomicMax(&out[1], (unsigned long long)__double_as_longlong(m));
    }
}

void launch_sweep5(int kind, bool impact, int64_t N, const uint32_t *order, const double4 *pos, const double4 *vin,
                   const double4 *win, double4 *vout, double4 *wout, const uint32_t *inc_start, const uint2 *inc,
                   const double *cb, const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out,
                   const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    const unsigned nb = (unsigned)((N + T5 - 1) / T5);
#define ARGS_PPT N, order, pos, vin, win, vout, wout, inc_start, inc, cb, Pa_in, Pb_in, Pa_out, Pb_out, bnd, sp
#define ARGS_TILE N, pos, vin, win, vout, wout, inc_start, inc, cb, Pa_in, Pb_in, Pa_out, Pb_out, bnd, sp
    if (kind == SWEEP5_PPT) {
        if (impact) k_sweep5_ppt<true, false><<<nb, T5, 0, s>>>(ARGS_PPT);
        else k_sweep5_ppt<false, false><<<nb, T5, 0, s>>>(ARGS_PPT);
    } else if (kind == SWEEP5_PPT_PF) {
        if (impact) k_sweep5_ppt<true, true><<<nb, T5, 0, s>>>(ARGS_PPT);
        else k_sweep5_ppt<false, true><<<nb, T5, 0, s>>>(ARGS_PPT);
    } else {
        if (impact) k_sweep5_tile<true><<<nb, T5, 0, s>>>(ARGS_TILE);
        else k_sweep5_tile<false><<<nb, T5, 0, s>>>(ARGS_TILE);
    }
#undef ARGS_PPT
#undef ARGS_TILE
}

void launch_row_bias(int64_t nc, const R4 *row, double *cb, cudaStream_t s)
{ if (nc) k_row_bias<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, row, cb); }

void launch_maxdiff(int64_t N, const double4 *a, const double4 *b, unsigned long long *out, cudaStream_t s)
{
    cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), s);
    if (N) k_maxdiff<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, a, b, out);
}
