// sweep_t2.cu -- the tile sweep (k_sweep_tile's work split and deterministic segmented
// reduction) with its memory traffic shaped for the L1 data pipe, which ncu showed to be the
// limiter of the sweep (l1tex__data_pipe_lsu_wavefronts ~86 % of peak):
//   * every 32-byte record (state double4, normals, rows) moves with ONE 256-bit access per
//     lane (LDG.E.256 / STG.E.256) instead of two 128-bit ones;
//   * the staged tile state lives in shared memory as double2 halves (16-byte lane stride:
//     no bank conflicts for LDS.128);
//   * the partner's state is loaded into registers explicitly (shared or global), not through
//     a generic pointer.
#include "common.cuh"
#include "kernels.h"
#include "sweep_core.cuh"

#ifndef SWEEPT2_MINB
#define SWEEPT2_MINB 5
#endif
constexpr int TT = 128;
constexpr int NWT = TT / 32;

__device__ __forceinline__ double4 cat2(const double2 a, const double2 b) { return make_double4(a.x, a.y, b.x, b.y); }

__global__ void __launch_bounds__(TT, SWEEPT2_MINB)
    k_sweep_t2(int64_t N, const double4 *__restrict__ vin, const double4 *__restrict__ win, double4 *__restrict__ vout,
               double4 *__restrict__ wout, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
               const G4 *__restrict__ geo, const R4 *__restrict__ row, const P4 *__restrict__ Pa_in,
               const P4 *__restrict__ Pb_in, P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out,
               const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    __shared__ double2 sVa[TT], sVb[TT], sWa[TT], sWb[TT];
    __shared__ double sAcc[NWT][6][32];
    __shared__ uint8_t sOwn[NWT][32];
    __shared__ uint32_t sI[TT + 1];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * TT;
    const int np = (int)min((int64_t)TT, N - p0);
    if (t < np) {
        const double4 v = ld4g(&vin[p0 + t]), o = ld4g(&win[p0 + t]);
        sVa[t] = make_double2(v.x, v.y); sVb[t] = make_double2(v.z, v.w);
        sWa[t] = make_double2(o.x, o.y); sWb[t] = make_double2(o.z, o.w);
    }
    for (int q = t; q <= np; q += TT) sI[q] = inc_start[p0 + q];
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
                const uint32_t c = ent.x & ~B_SIDE;
                const bool isB = (ent.x & B_SIDE) != 0;
                const uint32_t p = ent.y;
                const G4 g = ld4g(&geo[c]);
                const R4 rw = ld4g(&row[c]);
                const P4 pa = Pa_in[c], pb = Pb_in[c];
                double4 VP, WP;
                double mt = sp.mu_t;
                if (!(p & PARTNER_EXT)) {
                    const int64_t pl = (int64_t)p - p0;
                    if (pl >= 0 && pl < np) { VP = cat2(sVa[pl], sVb[pl]); WP = cat2(sWa[pl], sWb[pl]); }
                    else { VP = ld4g(&vin[p]); WP = ld4g(&win[p]); }
                } else {
                    d3 bv;
                    double mr;
                    boundary_body(p, bnd, bv, mt, mr);
                    VP = make_double4(bv.x, bv.y, bv.z, 0.0);
                    WP = make_double4(0.0, 0.0, 0.0, 0.0);
                }
                const double4 VS = cat2(sVa[o], sVb[o]), WS = cat2(sWa[o], sWb[o]);
                const HalfOut r = half_contact(isB ? VP : VS, isB ? WP : WS, isB ? VS : VP, isB ? WS : WP, isB, mt, g, rw,
                                               pa, pb, sp.rolling_dims);
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
        double4 V = cat2(sVa[me], sVb[me]), W = cat2(sWa[me], sWb[me]);
        const uint32_t cnt = e_me - s_me;
        if (cnt) {
            // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            V.x += im * sAcc[w][0][lane]; V.y += im * sAcc[w][1][lane]; V.z += im * sAcc[w][2][lane];
            W.x += iI * sAcc[w][3][lane]; W.y += iI * sAcc[w][4][lane]; W.z += iI * sAcc[w][5][lane];
        }
        st4g(&vout[p0 + me], V);
        st4g(&wout[p0 + me], W);
    }
}

void launch_sweep_t2(int64_t N, const double4 *vin, const double4 *win, double4 *vout, double4 *wout,
                     const uint32_t *inc_start, const uint2 *inc, const G4 *geo, const R4 *row, const P4 *Pa_in,
                     const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out, const DevBoundary *bnd, const SolveParams &sp,
                     cudaStream_t s)
{
    if (N) k_sweep_t2<<<(unsigned)((N + TT - 1) / TT), TT, 0, s>>>(N, vin, win, vout, wout, inc_start, inc, geo, row,
                                                                   Pa_in, Pb_in, Pa_out, Pb_out, bnd, sp);
}
