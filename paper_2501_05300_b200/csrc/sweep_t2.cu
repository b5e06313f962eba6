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
#define SWEEPT2_MINB 6
#endif
#ifndef SWEEPT2_TILE
#define SWEEPT2_TILE 128
#endif
constexpr int TT = SWEEPT2_TILE;   // particles per block tile (4 warps of 32 at the default)
constexpr int NWT = TT / 32;

__device__ __forceinline__ double4 cat2(const double2 a, const double2 b) { return make_double4(a.x, a.y, b.x, b.y); }

// ------------------------------------------------------------------ packed incidence
// Canonical reduction (trajectories bit-identical for any number of slabs).  The
// warp's segmented scan sums a particle's contributions with a tree that depends only on the
// particle's own list -- as long as the list does not straddle a 32-entry chunk boundary.  Once
// per step each warp's 32 particles are packed (first fit decreasing) into 32-lane chunks so that no list of
// <= 32 half-contacts straddles a boundary and a longer list starts on one (its pieces are then
// cut at fixed offsets 32, 64, ... of its own list); unused lanes are holes (0xFFFFFFFF).  The
// packing depends only on list lengths, the sums only on the lists (ordered by partner gid), so
// every decomposition and warp grouping produces the same bits.
constexpr uint32_t PK_HOLE = 0xFFFFFFFFu;
thread_local bool g_t2_rows_by_contact = false;   // diagnostic variant flags, per host thread
thread_local bool g_t2_stage = false;
thread_local int g_t2_exp = 0;

// one warp per 32 consecutive particles (the sweep's warp grouping): first-fit packing
__global__ void k_pack_plan(int64_t N, const uint32_t *__restrict__ inc_start, uint32_t *__restrict__ off_local,
                            uint32_t *__restrict__ wsize)
{
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (32 * g >= N) return;                               // whole warp
    const int64_t i = 32 * g + lane;
    const uint32_t L = i < N ? inc_start[i + 1] - inc_start[i] : 0u;
    uint32_t my_off = 0, cap = 0, binno = 0;               // lane s: open slot s (capacity, bin)
    uint32_t nb = 0, nslots = 0;
    unsigned longs = __ballot_sync(0xffffffffu, L > 32u);
    while (longs) {                                        // lists > 32 start on a chunk boundary
        const int p = __ffs(longs) - 1;
        const uint32_t Lp = __shfl_sync(0xffffffffu, L, p);
        if (lane == p) my_off = 32u * nb;
        nb += Lp / 32u;
        if (Lp % 32u) {
            if (lane == (int)nslots) { cap = 32u - Lp % 32u; binno = nb; }
            nslots++;
            nb++;
        }
        longs &= longs - 1;
    }
    // first fit decreasing: lists by decreasing length (ties: particle order) into the first
    // open chunk with room -- close to the fewest chunks, so few holes
    for (uint32_t Lc = 32u; Lc >= 1u; Lc--) {
    unsigned shorts = __ballot_sync(0xffffffffu, L == Lc);
    while (shorts) {
        const int p = __ffs(shorts) - 1;
        const uint32_t Lp = __shfl_sync(0xffffffffu, L, p);
        const unsigned fit = __ballot_sync(0xffffffffu, lane < (int)nslots && cap >= Lp);
        uint32_t off;
        if (fit) {
            const int sl = __ffs(fit) - 1;
            const uint32_t c = __shfl_sync(0xffffffffu, cap, sl), b = __shfl_sync(0xffffffffu, binno, sl);
            off = 32u * b + (32u - c);
            if (lane == sl) cap -= Lp;
        } else {
            off = 32u * nb;
            if (lane == (int)nslots) { cap = 32u - Lp; binno = nb; }
            nslots++;
            nb++;
        }
        if (lane == p) my_off = off;
        shorts &= shorts - 1;
    }
    }
    if (i < N) off_local[i] = my_off;
    if (lane == 0) wsize[g] = 32u * nb;
}

__global__ void k_pack_fill(int64_t N, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                            const uint32_t *__restrict__ off_local, const uint32_t *__restrict__ wbase,
                            uint32_t *__restrict__ pstart, uint2 *__restrict__ pinc)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t ps = wbase[i >> 5] + off_local[i], s = inc_start[i], e = inc_start[i + 1];
    pstart[i] = ps;
    for (uint32_t k = s; k < e; k++) pinc[ps + (k - s)] = inc[k];
}

// packed size of the whole bed (host reads it to size pinc), then the fill
void pack_plan(int64_t N, const uint32_t *inc_start, uint32_t *off_local, uint32_t *wsize, uint32_t *wbase,
               void *scan_tmp, cudaStream_t s, long long *launches)
{
    const int64_t nw = (N + 31) / 32;
    if (nw) k_pack_plan<<<(unsigned)((nw + 3) / 4), 128, 0, s>>>(N, inc_start, off_local, wsize);
    scan_u32(wsize, wbase, nw, scan_tmp, s, launches);
    *launches += 1;
}
void pack_fill(int64_t N, const uint32_t *inc_start, const uint2 *inc, const uint32_t *off_local, const uint32_t *wbase,
               uint32_t *pstart, uint2 *pinc, int64_t npacked, cudaStream_t s, long long *launches)
{
    if (npacked) cudaMemsetAsync(pinc, 0xFF, npacked * sizeof(uint2), s);
    if (N) k_pack_fill<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, inc_start, inc, off_local, wbase, pstart, pinc);
    *launches += 1;
}

// per step (and per stage): normals and rows gathered into packed order, both halves a copy
__global__ void k_pack_rows(int64_t np, const uint2 *__restrict__ pinc, const G4 *__restrict__ geo,
                            const R4 *__restrict__ row, G4 *__restrict__ gpk, R4 *__restrict__ rpk)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= np) return;
    const uint32_t e = pinc[k].x;
    if (e == PK_HOLE) return;
    const uint32_t c = e & INC_CMASK;
    if (gpk) st4g(&gpk[k], ld4g(&geo[c]));
    st4g(&rpk[k], ld4g(&row[c]));
}
__global__ void k_p8_pack(int64_t nc, const P4 *__restrict__ a, const P4 *__restrict__ b, P8 *__restrict__ o)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nc) stP8(&o[c], a[c], b[c]);
}
__global__ void k_p8_unpack(int64_t nc, const P8 *__restrict__ q, P4 *__restrict__ a, P4 *__restrict__ b)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const P8 v = ldP8(&q[c]);
    a[c] = v.a;
    b[c] = v.b;
}
void pack_rows(int64_t np, const uint2 *pinc, const G4 *geo, const R4 *row, G4 *gpk, R4 *rpk, cudaStream_t s)
{ if (np) k_pack_rows<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(np, pinc, geo, row, gpk, rpk); }
void p8_pack(int64_t nc, const P4 *a, const P4 *b, P8 *o, cudaStream_t s)
{ if (nc) k_p8_pack<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, a, b, o); }
void p8_unpack(int64_t nc, const P8 *q, P4 *a, P4 *b, cudaStream_t s)
{ if (nc) k_p8_unpack<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, q, a, b); }

// PACKED: the canonical reduction above (default); false: the contiguous CSR chunks (fastest
// layout-independent of packing; bit-reproducible run to run but rounding depends on the warp
// grouping, i.e. on the decomposition)
// EXP (timing experiments on the shipped kernel, dem_bench_sweeps 44/45): 1 the contact
// arithmetic replaced by a few additions of its inputs (memory side only), 2 the contact records
// and impulses not loaded (arithmetic on constants)
__device__ __forceinline__ HalfOut t2_fake(const double4 VA, const double4 WA, const double4 VB, const double4 WB,
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

// ---- one-chunk-ahead TMA staging (STG): the chunk's packed incidence, normals and rows are
// contiguous (1 KB + 1 KB + 256 B), so one lane per warp moves them with 1D bulk copies
// (cp.async.bulk, completion on an mbarrier) into a two-slot ring while the warp computes the
// previous chunk: no registers held for the prefetch, no LSU instructions for the records.
constexpr int STG_BYTES = 32 * (int)sizeof(G4) + 32 * (int)sizeof(R4) + 32 * (int)sizeof(uint2);
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
struct __align__(128) StgSlot { G4 g[32]; R4 r[32]; uint2 e[32]; };
__device__ __forceinline__ void stg_issue(StgSlot *sl, uint64_t *bar, const G4 *geo, const R4 *row, const uint2 *inc,
                                          uint32_t kb)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads of the slot before the refill
    mbar_expect_tx(bar, STG_BYTES);
    bulk_g2s(sl->g, geo + kb, 32 * sizeof(G4), bar);
    bulk_g2s(sl->r, row + kb, 32 * sizeof(R4), bar);
    bulk_g2s(sl->e, inc + kb, 32 * sizeof(uint2), bar);
}
// a staged chunk's records are stored as two planes (x,y of the 32 lanes, then z,w): each
// LDS.128 of the warp then reads 512 contiguous bytes, conflict-free
__device__ __forceinline__ double4 lds_plane(const double4 *base, int lane)
{
    const double2 *p = reinterpret_cast<const double2 *>(base);
    const double2 a = p[lane], b = p[32 + lane];
    return make_double4(a.x, a.y, b.x, b.y);
}
__global__ void k_to_planes(int64_t np, const double4 *__restrict__ in, double2 *__restrict__ out)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= np) return;
    const double4 v = in[k];
    const int64_t c = k >> 5, l = k & 31;
    out[64 * c + l] = make_double2(v.x, v.y);
    out[64 * c + 32 + l] = make_double2(v.z, v.w);
}
void to_planes(int64_t np, const double4 *in, double4 *out, cudaStream_t s)
{ if (np) k_to_planes<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(np, in, reinterpret_cast<double2 *>(out)); }

template <bool PACKED, bool ROWS_PK = true, int EXP = 0, bool STG = false>
__global__ void __launch_bounds__(TT, SWEEPT2_MINB)
    k_sweep_t2(int64_t N, const double4 *__restrict__ vin, const double4 *__restrict__ win, double4 *__restrict__ vout,
               double4 *__restrict__ wout, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
               const uint32_t *__restrict__ pstart, const uint32_t *__restrict__ wbase,
               const G4 *__restrict__ geo, const R4 *__restrict__ row, const P4 *__restrict__ Pa_in,
               const P4 *__restrict__ Pb_in, P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out,
               const P8 *__restrict__ P8_in, P8 *__restrict__ P8_out, const DevBoundary *__restrict__ bnd,
               SolveParams sp)
{
    __shared__ double2 sVa[TT], sVb[TT], sWa[TT], sWb[TT];
    __shared__ double sAcc[NWT][6][32];
    __shared__ uint8_t sOwn[NWT][32];
    __shared__ uint32_t sI[TT + 1];
    __shared__ uint32_t sPS[PACKED ? TT : 1];
    __shared__ StgSlot sStg[STG ? NWT : 1][STG ? 2 : 1];
    __shared__ uint64_t sBar[NWT][2];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (STG && lane == 0) {
        mbar_init(&sBar[w][0], 1);
        mbar_init(&sBar[w][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int64_t p0 = (int64_t)blockIdx.x * TT;
    const int np = (int)min((int64_t)TT, N - p0);
    if (t < np) {
        const double4 v = ld4g(&vin[p0 + t]), o = ld4g(&win[p0 + t]);
        sVa[t] = make_double2(v.x, v.y); sVb[t] = make_double2(v.z, v.w);
        sWa[t] = make_double2(o.x, o.y); sWb[t] = make_double2(o.z, o.w);
    }
    for (int q = t; q <= np; q += TT) sI[q] = inc_start[p0 + q];
    if (PACKED && t < np) sPS[t] = pstart[p0 + t];
#pragma unroll
    for (int f = 0; f < 6; f++) sAcc[w][f][lane] = 0.0;
    __syncthreads();
    const int lo_p = 32 * w, hi_p = min(32 * w + 32, np);
    const int me = lo_p + lane;
    const uint32_t cnt_me = me < hi_p ? sI[me + 1] - sI[me] : 0u;
    const uint32_t s_me = me < hi_p ? (PACKED ? sPS[me] : sI[me]) : 0u, e_me = s_me + cnt_me;
    if (lo_p < np) {
        const uint32_t k0 = PACKED ? wbase[(p0 >> 5) + w] : sI[lo_p];
        const uint32_t k1 = PACKED ? wbase[(p0 >> 5) + w + 1] : sI[hi_p];
        uint2 ent_next = make_uint2(0, 0);
        if (STG) {
            if (lane == 0) {
                stg_issue(&sStg[w][0], &sBar[w][0], geo, row, inc, k0);
                if (k0 + 32 < k1) stg_issue(&sStg[w][1], &sBar[w][1], geo, row, inc, k0 + 32);
            }
        } else if (k0 + lane < k1) ent_next = inc[k0 + lane];
        int carry = 0;
        uint32_t it = 0;
        for (uint32_t kb = k0; kb < k1; kb += 32, it++) {
            const uint32_t k = kb + lane;
            uint2 ent = ent_next;
            G4 gs;
            R4 rs;
            if (STG) {
                // chunk it sits in slot it & 1, filled for the (it >> 1)-th time
                StgSlot *sl = &sStg[w][it & 1];
                mbar_wait(&sBar[w][it & 1], (it >> 1) & 1u);
                ent = sl->e[lane];
                if (ent.x != PK_HOLE) { gs = lds_plane(sl->g, lane); rs = lds_plane(sl->r, lane); }
                __syncwarp();
                if (lane == 0 && kb + 64 < k1) stg_issue(sl, &sBar[w][it & 1], geo, row, inc, kb + 64);
            }
            const bool valid = k < k1 && (!PACKED || ent.x != PK_HOLE);
            if (!STG && kb + 32 + lane < k1) ent_next = inc[kb + 32 + lane];
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
                // PACKED: normals and rows duplicated per half-contact in packed order (coalesced),
                // both impulse records of the contact in one 32-byte slot
                G4 g;
                R4 rw;
                P4 pa, pb;
                if (EXP == 2) {
                    g = mkG4(0.6, 0.0, 0.8, 1e-4); rw = mkR4(1e-3, 1e-3, 1e-3, 1e-3);
                    pa = mkP4(1e-6, 0, 0, 0); pb = mkP4(0, 0, 0, 0);
                } else {
                    if (STG) { g = gs; rw = rs; }
                    else {
                        g = ld4g(PACKED && ROWS_PK ? &geo[k] : &geo[c]);
                        rw = ld4g(PACKED && ROWS_PK ? &row[k] : &row[c]);
                    }
                    if (PACKED) { const P8 q = ldP8(&P8_in[c]); pa = q.a; pb = q.b; }
                    else { pa = Pa_in[c]; pb = Pb_in[c]; }
                }
                // operands in the canonical (a, b) order.  Particle pairs: bodies a and b are
                // loaded by index straight into their slots (shared memory inside the tile, else
                // global), so no per-value selects between self and partner (measured: same
                // time as the load-then-select form, bit-identical); boundary partners are body b.
                double4 VA, WA, VB, WB;
                double mt = sp.mu_t;
                if (!(p & PARTNER_EXT)) {
                    const int64_t ga = isB ? (int64_t)p : p0 + o, gb = isB ? p0 + o : (int64_t)p;
                    const int64_t la = ga - p0, lb = gb - p0;
                    if (la >= 0 && la < np) { VA = cat2(sVa[la], sVb[la]); WA = cat2(sWa[la], sWb[la]); }
                    else { VA = ld4g(&vin[ga]); WA = ld4g(&win[ga]); }
                    if (lb >= 0 && lb < np) { VB = cat2(sVa[lb], sVb[lb]); WB = cat2(sWa[lb], sWb[lb]); }
                    else { VB = ld4g(&vin[gb]); WB = ld4g(&win[gb]); }
                } else {
                    d3 bv;
                    double mr;
                    boundary_body(p, bnd, bv, mt, mr);
                    VA = cat2(sVa[o], sVb[o]);
                    WA = cat2(sWa[o], sWb[o]);
                    VB = make_double4(bv.x, bv.y, bv.z, 0.0);
                    WB = make_double4(0.0, 0.0, 0.0, 0.0);
                }
                const HalfOut r = EXP == 1 ? t2_fake(VA, WA, VB, WB, g, rw, pa, pb)
                                           : half_contact(VA, WA, VB, WB, isB, mt, g, rw, pa, pb, sp.rolling_dims);
                if (!isB) {   // both halves compute the same impulses; body a stores them
                    if (PACKED) stP8(&P8_out[c], r.Pa, r.Pb);
                    else { Pa_out[c] = r.Pa; Pb_out[c] = r.Pb; }
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
            // holes only trail a chunk: a segment also ends before the first hole
            const unsigned vmask = PACKED ? __ballot_sync(0xffffffffu, valid) : 0xffffffffu;
            const bool seg_end = valid && (lane == 31 || ((smask >> (lane + 1)) & 1u) || k + 1 >= k1 ||
                                           (PACKED && !((vmask >> (lane + 1)) & 1u)));
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
        const uint32_t cnt = cnt_me;
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
                     const uint32_t *inc_start, const uint2 *inc, const PackedInc *pk, const G4 *geo, const R4 *row,
                     const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out, const DevBoundary *bnd,
                     const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    const unsigned gb = (unsigned)((N + TT - 1) / TT);
    if (pk && g_t2_exp) {             // diagnostic (dem_bench_sweeps 44/45): timing experiments
        if (g_t2_exp == 1)
            k_sweep_t2<true, true, 1><<<gb, TT, 0, s>>>(N, vin, win, vout, wout, inc_start, pk->inc, pk->start, pk->wbase,
                                                        pk->geo, pk->row, nullptr, nullptr, nullptr, nullptr, pk->p8in,
                                                        pk->p8out, bnd, sp);
        else
            k_sweep_t2<true, true, 2><<<gb, TT, 0, s>>>(N, vin, win, vout, wout, inc_start, pk->inc, pk->start, pk->wbase,
                                                        pk->geo, pk->row, nullptr, nullptr, nullptr, nullptr, pk->p8in,
                                                        pk->p8out, bnd, sp);
        return;
    }
    if (pk && g_t2_stage)             // dem_bench_sweeps 9: TMA-staged records
        k_sweep_t2<true, true, 0, true><<<gb, TT, 0, s>>>(N, vin, win, vout, wout, inc_start, pk->inc, pk->start,
                                                          pk->wbase, pk->geo, pk->row, nullptr, nullptr, nullptr, nullptr,
                                                          pk->p8in, pk->p8out, bnd, sp);
    else if (pk && g_t2_rows_by_contact)   // diagnostic (dem_bench_sweeps 8): contact-indexed rows
        k_sweep_t2<true, false><<<gb, TT, 0, s>>>(N, vin, win, vout, wout, inc_start, pk->inc, pk->start, pk->wbase,
                                                  pk->geo, pk->row, nullptr, nullptr, nullptr, nullptr, pk->p8in,
                                                  pk->p8out, bnd, sp);
    else if (pk)
        k_sweep_t2<true><<<gb, TT, 0, s>>>(N, vin, win, vout, wout, inc_start, pk->inc, pk->start, pk->wbase, pk->geo,
                                           pk->row, nullptr, nullptr, nullptr, nullptr, pk->p8in, pk->p8out, bnd, sp);
    else
        k_sweep_t2<false><<<gb, TT, 0, s>>>(N, vin, win, vout, wout, inc_start, inc, nullptr, nullptr, geo, row, Pa_in,
                                            Pb_in, Pa_out, Pb_out, nullptr, nullptr, bnd, sp);
}

// ==================================================================== layout experiment (t3)
// The t2 kernel with (P8) the two impulse records of a contact interleaved in one 32-byte slot
// (one 256-bit load and store instead of two 128-bit ones) and (VW) a particle's v and w
// interleaved in one 64-byte record (both gathers hit one cache line).  Diagnostic only: the
// bench converts the layouts before timing (dem_bench_sweeps variants 60-63).
struct __align__(32) VW { double4 v, w; };

template <bool USE_P8, bool USE_VW, bool NOSEL = false>
__global__ void __launch_bounds__(TT, SWEEPT2_MINB)
    k_sweep_t3(int64_t N, const double4 *__restrict__ vin, const double4 *__restrict__ win, double4 *__restrict__ vout,
               double4 *__restrict__ wout, const VW *__restrict__ vwin, VW *__restrict__ vwout,
               const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc, const G4 *__restrict__ geo,
               const R4 *__restrict__ row, const P4 *__restrict__ Pa_in, const P4 *__restrict__ Pb_in,
               P4 *__restrict__ Pa_out, P4 *__restrict__ Pb_out, const P8 *__restrict__ P8in, P8 *__restrict__ P8out,
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
        double4 v, o;
        if (USE_VW) { v = ld4g(&vwin[p0 + t].v); o = ld4g(&vwin[p0 + t].w); }
        else { v = ld4g(&vin[p0 + t]); o = ld4g(&win[p0 + t]); }
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
                const uint32_t c = ent.x & INC_CMASK;
                const bool isB = (ent.x & B_SIDE) != 0;
                const uint32_t p = ent.y;
                const G4 g = ld4g(&geo[c]);
                const R4 rw = ld4g(&row[c]);
                P4 pa, pb;
                if (USE_P8) { const P8 q = ldP8(&P8in[c]); pa = q.a; pb = q.b; }
                else { pa = Pa_in[c]; pb = Pb_in[c]; }
                double4 VP, WP;
                double mt = sp.mu_t;
                if (!(p & PARTNER_EXT)) {
                    const int64_t pl = (int64_t)p - p0;
                    if (pl >= 0 && pl < np) { VP = cat2(sVa[pl], sVb[pl]); WP = cat2(sWa[pl], sWb[pl]); }
                    else if (USE_VW) { VP = ld4g(&vwin[p].v); WP = ld4g(&vwin[p].w); }
                    else { VP = ld4g(&vin[p]); WP = ld4g(&win[p]); }
                } else {
                    d3 bv;
                    double mr;
                    boundary_body(p, bnd, bv, mt, mr);
                    VP = make_double4(bv.x, bv.y, bv.z, 0.0);
                    WP = make_double4(0.0, 0.0, 0.0, 0.0);
                }
                const double4 VS = cat2(sVa[o], sVb[o]), WS = cat2(sWa[o], sWb[o]);
                const HalfOut r = NOSEL ? half_contact(VS, WS, VP, WP, isB, mt, g, rw, pa, pb, sp.rolling_dims)
                                        : half_contact(isB ? VP : VS, isB ? WP : WS, isB ? VS : VP, isB ? WS : WP, isB, mt,
                                                       g, rw, pa, pb, sp.rolling_dims);
                if (!isB) {
                    if (USE_P8) stP8(&P8out[c], r.Pa, r.Pb);
                    else { Pa_out[c] = r.Pa; Pb_out[c] = r.Pb; }
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
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            V.x += im * sAcc[w][0][lane]; V.y += im * sAcc[w][1][lane]; V.z += im * sAcc[w][2][lane];
            W.x += iI * sAcc[w][3][lane]; W.y += iI * sAcc[w][4][lane]; W.z += iI * sAcc[w][5][lane];
        }
        if (USE_VW) { st4g(&vwout[p0 + me].v, V); st4g(&vwout[p0 + me].w, W); }
        else { st4g(&vout[p0 + me], V); st4g(&wout[p0 + me], W); }
    }
}

__global__ void k_pack_p8(int64_t nc, const P4 *__restrict__ a, const P4 *__restrict__ b, P8 *__restrict__ o)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nc) { o[c].a = a[c]; o[c].b = b[c]; }
}
__global__ void k_pack_vw(int64_t n, const double4 *__restrict__ v, const double4 *__restrict__ w, VW *__restrict__ o,
                          double4 *__restrict__ vback)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (vback) { vback[i] = o[i].v; return; }     // unpack direction: v of VW -> vback
    o[i].v = v[i];
    o[i].w = w[i];
}

// t3 experiment driver: n sweeps from (vin, win, Pa, Pb); the final v written back to vres
void run_sweep_t3(int variant, int n, int64_t N, int64_t nc, const double4 *vin, const double4 *win, double4 *vbuf[2],
                  double4 *wbuf[2], const uint32_t *inc_start, const uint2 *inc, const G4 *geo, const R4 *row,
                  P4 *Pa[2], P4 *Pb[2], void *scratch, const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s,
                  double4 *vres, cudaEvent_t e0, cudaEvent_t e1)
{
    const bool p8 = variant & 1, vw = (variant >> 1) & 1, nosel = (variant >> 2) & 1;
    P8 *q[2] = {(P8 *)scratch, (P8 *)scratch + nc};
    VW *u[2] = {(VW *)(q[1] + nc), (VW *)(q[1] + nc) + N};
    const unsigned gb = (unsigned)((N + TT - 1) / TT);
    k_pack_p8<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, Pa[0], Pb[0], q[0]);
    k_pack_vw<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, vin, win, u[0], nullptr);
    cudaEventRecord(e0, s);
    const double4 *vi = vin, *wi = win;
    for (int it = 0; it < n; it++) {
        const int a = it & 1, b = a ^ 1;
#define T3ARGS N, vi, wi, vbuf[a], wbuf[a], u[a], u[b], inc_start, inc, geo, row, Pa[a], Pb[a], Pa[b], Pb[b], q[a], q[b], bnd, sp
        if (nosel) k_sweep_t3<true, false, true><<<gb, TT, 0, s>>>(T3ARGS);   // timing only: wrong orientation for B
        else if (p8 && vw) k_sweep_t3<true, true><<<gb, TT, 0, s>>>(T3ARGS);
        else if (p8) k_sweep_t3<true, false><<<gb, TT, 0, s>>>(T3ARGS);
        else if (vw) k_sweep_t3<false, true><<<gb, TT, 0, s>>>(T3ARGS);
        else k_sweep_t3<false, false><<<gb, TT, 0, s>>>(T3ARGS);
#undef T3ARGS
        vi = vbuf[a]; wi = wbuf[a];
    }
    cudaEventRecord(e1, s);
    const int last = (n - 1) & 1;
    if (vw) k_pack_vw<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, nullptr, nullptr, u[last ^ 1], vres);
    else cudaMemcpyAsync(vres, vbuf[last], N * sizeof(double4), cudaMemcpyDeviceToDevice, s);
}
