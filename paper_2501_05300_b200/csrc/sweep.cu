// sweep.cu -- the projected Jacobi impulse sweep (P:115-125 under SPOOK, P:132-134;
// readings R2, R4, R7-R10), the method's hot loop: N_it (+ N_imp) launches per time step.
//
// Contact-once tiles.  A CTA owns a tile of TT consecutive particles of the rebuild's (level,
// Morton) order.  Every contact is an "item" of the tile that owns one of its bodies:
//   * intra-tile particle pairs: ONE item, owned by body a; its body-b contribution goes to a
//     shared-memory slot of body b (slots of a particle are contiguous);
//   * cross-tile particle pairs: one item in each of the two tiles (each evaluates the contact
//     from the same canonical operands, bit-identically; each keeps only its own body's share);
//   * wall / plate contacts: one item, owned by the particle.
// A tile's items are stored contiguously, grouped by owner (warp w's 32 particles' items form
// one range), so records move with coalesced 256-bit accesses:
//   CRec 32 B per item: n (a -> b; two fp64 components, the third reconstructed), delta and the
//        stage's SPOOK bias b (fp64)
//   PRec 32 B per item: P_n, P_t (3), P_r (3) and a 32-bit meta word (partner, flags); storage
//        precision SWEEP_PMODE (kernels.h)
// Everything else the contact row needs is derived from the radii: R* = r_a r_b/(r_a + r_b),
// l_a = r_a - delta/2, l_b = r_b - delta/2, mu_r R*, Sigma-hat = Cs / sqrt(2 R* delta) (R4).
//
// Reduction (deterministic, decomposition-invariant, no float atomics).  Each body's share of a
// contact increment is converted to int64 fixed point with a power-of-two scale chosen from the
// body's own mass-splitting weight (c/m, c/I) and summed exactly; integer sums are order-free,
// so a particle's velocity update does not depend on how contacts fall into tiles, warps or
// ranks: trajectories are bit-identical for any decomposition.  Resolution
// ~2^-48 m/s (linear) and ~2^-44 rad/s (angular) of velocity per contribution, far below the
// fp32 impulse storage's rounding; a contribution beyond 2^56 units (~256 m/s or 4096 rad/s per
// sweep) or a non-finite one poisons the particle's velocity with NaN (the step rolls back).
#include "common.cuh"
#include "kernels.h"
#include "sweep_core.cuh"

constexpr int TT = SWEEP_TILE;           // particles per tile (one CTA), kernels.h
constexpr int NWT = TT / 32;
constexpr int SLOT_CAP = SWEEP_SLOT_CAP; // intra-tile body-b slots per tile
constexpr int FX_EL = 48, FX_EA = 44;    // fixed-point exponents (linear, angular)

__device__ __forceinline__ double4 cat2(const double2 a, const double2 b) { return make_double4(a.x, a.y, b.x, b.y); }

// ------------------------------------------------------------------ fixed point
// Scale of body i: 2^(E + ilogb(w_i) - floor(log2 c_i)) ~ 2^E m_i (w = c/m, c = contact count;
// likewise with c/I): integer units of 2^-E m/s (rad/s) of velocity, whatever the particle size.
__device__ __forceinline__ int fx_exp(double w, uint32_t c)
{
    return (int)((__double_as_longlong(w) >> 52) & 0x7FF) - 1023 - (31 - __clz((int)c));
}
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }
// Fixed-point value of x s (s a power of two, so x s is exact), kept as raw bits: t = x s + 1.5 2^52
// rounds x s to an integer exactly (RN-even, like llrint) whenever |x s| <= 2^51, and then the
// bit pattern of t is round(x s) + FX_MAGIC_BITS.  Sums of raw patterns are taken mod 2^64 and
// the c FX_MAGIC_BITS are subtracted once per particle (exact: integer arithmetic wraps).  fx1
// returns the deviation of t's exponent field from 0x433 (nonzero: out of range or NaN -> the
// slow path, which produces the same raw form).
constexpr double FX_MAGIC = 6755399441055744.0;            // 1.5 2^52
constexpr long long FX_MAGIC_BITS = 0x4338000000000000LL;
struct Fx6 { long long v[6]; };
__device__ __forceinline__ unsigned fx1(double x, double s, long long &o)
{
    o = __double_as_longlong(__fma_rn(x, s, FX_MAGIC));
    return ((unsigned)((unsigned long long)o >> 52)) ^ 0x433u;
}
__device__ __noinline__ Fx6 fx6_slow(const d3 L, const d3 A, double sL, double sA, bool &bad)
{
    const double y[6] = {L.x * sL, L.y * sL, L.z * sL, A.x * sA, A.y * sA, A.z * sA};
    Fx6 o;
    for (int f = 0; f < 6; f++) {
        if (!(fabs(y[f]) < 72057594037927936.0)) { bad = true; o.v[f] = FX_MAGIC_BITS; }   // >= 2^56 or NaN
        else o.v[f] = (long long)((unsigned long long)__double2ll_rn(y[f]) + (unsigned long long)FX_MAGIC_BITS);
    }
    return o;
}
__device__ __forceinline__ Fx6 fx6(const d3 L, const d3 A, double sL, double sA, bool &bad)
{
    Fx6 o;
    const unsigned e = fx1(L.x, sL, o.v[0]) | fx1(L.y, sL, o.v[1]) | fx1(L.z, sL, o.v[2]) | fx1(A.x, sA, o.v[3]) |
                       fx1(A.y, sA, o.v[4]) | fx1(A.z, sA, o.v[5]);
    if (e) o = fx6_slow(L, A, sL, sA, bad);
    return o;
}
// angular shares with one fixed rounding sequence (every path that produces a body's share of a
// contact must give the same bits): body a -(l_a n x dPt + dPr), body b -l_b n x dPt + dPr
__device__ __forceinline__ d3 share_a(double la, const d3 x, const d3 r)
{
    return mk(-__fma_rn(la, x.x, r.x), -__fma_rn(la, x.y, r.y), -__fma_rn(la, x.z, r.z));
}
__device__ __forceinline__ d3 share_b(double lb, const d3 x, const d3 r)
{
    return mk(__fma_rn(-lb, x.x, r.x), __fma_rn(-lb, x.y, r.y), __fma_rn(-lb, x.z, r.z));
}

// ------------------------------------------------------------------ contact record (CRec)
// n is stored as two fp64 components; the third, the largest in magnitude (>= 1/sqrt 3), is
// sqrt(1 - u^2 - v^2) with its axis and sign in the low 3 mantissa bits of delta (delta itself
// is used with those bits cleared: <= 7 ulp).  SWEEP_PMODE 1 also keeps the item's meta word in
// the low 16 bits of u and v (n then carries ~36 bits: 1e-11, against 6e-8 of fp32 normals).
#if SWEEP_PMODE == 1
constexpr unsigned long long N_LOWMASK = 0xFFFFull;
#else
constexpr unsigned long long N_LOWMASK = 0ull;
#endif
__device__ __forceinline__ void crec_decode(const double4 c, d3 &n, double &delta, double &b)
{
    const unsigned long long db = (unsigned long long)__double_as_longlong(c.z);
    delta = __longlong_as_double((long long)(db & ~7ull));
    b = c.w;
    const double u = __longlong_as_double((long long)((unsigned long long)__double_as_longlong(c.x) & ~N_LOWMASK));
    const double v = __longlong_as_double((long long)((unsigned long long)__double_as_longlong(c.y) & ~N_LOWMASK));
    const double s = __fma_rn(-u, u, __fma_rn(-v, v, 1.0));
    double m = s * rsqrt64(s);
    if (db & 4ull) m = -m;
    const int ax = (int)(db & 3ull);
    n = ax == 0 ? mk(m, u, v) : (ax == 1 ? mk(v, m, u) : mk(u, v, m));
}
__device__ __forceinline__ double4 crec_encode(const d3 n, double delta, double b, uint32_t meta)
{
    const double ax0 = fabs(n.x), ax1 = fabs(n.y), ax2 = fabs(n.z);
    const int ax = (ax0 >= ax1 && ax0 >= ax2) ? 0 : (ax1 >= ax2 ? 1 : 2);
    const double big = ax == 0 ? n.x : (ax == 1 ? n.y : n.z);
    double u = ax == 0 ? n.y : (ax == 1 ? n.z : n.x), v = ax == 0 ? n.z : (ax == 1 ? n.x : n.y);
    if (N_LOWMASK) {
        u = __longlong_as_double((long long)(((unsigned long long)__double_as_longlong(u) & ~N_LOWMASK) | (meta & 0xFFFFu)));
        v = __longlong_as_double((long long)(((unsigned long long)__double_as_longlong(v) & ~N_LOWMASK) | (meta >> 16)));
    }
    const unsigned long long db = ((unsigned long long)__double_as_longlong(delta) & ~7ull) | (unsigned long long)ax |
                                  (big < 0.0 ? 4ull : 0ull);
    return make_double4(u, v, __longlong_as_double((long long)db), b);
}

// ------------------------------------------------------------------ impulse record (PRec)
// PMODE 0: P_n, P_t, P_r f32 + meta (32 B); 1: P_n f64, P_t, P_r f32 (32 B), meta in the CRec;
// 2: all f64 + meta (64 B, two PRec units).  The sweep rounds each new impulse to its storage
// precision and applies exactly the stored increments (momentum stays consistent).
#if SWEEP_PMODE == 0
typedef float PN_T;
typedef float PT_T;
struct PRaw { float4 a, b; };
#elif SWEEP_PMODE == 1
typedef double PN_T;
typedef float PT_T;
struct PRaw { double4 a; };
#else
typedef double PN_T;
typedef double PT_T;
struct PRaw { double4 a, b; };
#endif
__device__ __forceinline__ double4 ldg4d(const void *p)
{
    double4 v;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void stg4d(void *p, double a, double b, double c, double d)
{
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ double pk2(float x, float y)
{
    return __longlong_as_double((long long)(((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(x)));
}
__device__ __forceinline__ float lo2(double d) { return __uint_as_float((uint32_t)(unsigned long long)__double_as_longlong(d)); }
__device__ __forceinline__ float hi2(double d) { return __uint_as_float((uint32_t)((unsigned long long)__double_as_longlong(d) >> 32)); }

__device__ __forceinline__ PRaw ld_praw(const PRec *P, uint32_t k)
{
    PRaw r;
#if SWEEP_PMODE == 0
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y), "=f"(r.b.z), "=f"(r.b.w)
        : "l"(P + k));
#elif SWEEP_PMODE == 1
    r.a = ldg4d(P + k);
#else
    r.a = ldg4d(P + 2 * (size_t)k);
    r.b = ldg4d(reinterpret_cast<const double *>(P + 2 * (size_t)k) + 4);
#endif
    return r;
}
__device__ __forceinline__ uint32_t praw_meta(const PRaw &r, const double4 c)
{
#if SWEEP_PMODE == 0
    (void)c;
    return __float_as_uint(r.b.w);
#elif SWEEP_PMODE == 1
    (void)r;
    return (uint32_t)((unsigned long long)__double_as_longlong(c.x) & 0xFFFFull) |
           ((uint32_t)((unsigned long long)__double_as_longlong(c.y) & 0xFFFFull) << 16);
#else
    (void)c;
    return (uint32_t)(unsigned long long)__double_as_longlong(r.b.w);
#endif
}
__device__ __forceinline__ void praw_vals(const PRaw &r, double &pn, d3 &pt, d3 &pr)
{
#if SWEEP_PMODE == 0
    pn = r.a.x; pt = mk(r.a.y, r.a.z, r.a.w); pr = mk(r.b.x, r.b.y, r.b.z);
#elif SWEEP_PMODE == 1
    pn = r.a.x;
    pt = mk(lo2(r.a.y), hi2(r.a.y), lo2(r.a.z));
    pr = mk(hi2(r.a.z), lo2(r.a.w), hi2(r.a.w));
#else
    pn = r.a.x; pt = mk(r.a.y, r.a.z, r.a.w); pr = mk(r.b.x, r.b.y, r.b.z);
#endif
}
template <typename C>
__device__ __forceinline__ void st_prec(PRec *P, uint32_t k, const C &c, uint32_t meta)
{
#if SWEEP_PMODE == 0
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(P + k), "f"(c.pn), "f"(c.pt[0]),
                 "f"(c.pt[1]), "f"(c.pt[2]), "f"(c.pr[0]), "f"(c.pr[1]), "f"(c.pr[2]), "f"(__uint_as_float(meta))
                 : "memory");
#elif SWEEP_PMODE == 1
    (void)meta;
    stg4d(P + k, c.pn, pk2(c.pt[0], c.pt[1]), pk2(c.pt[2], c.pr[0]), pk2(c.pr[1], c.pr[2]));
#else
    double *q = reinterpret_cast<double *>(P + 2 * (size_t)k);
    stg4d(q, c.pn, c.pt[0], c.pt[1], c.pt[2]);
    stg4d(q + 4, c.pr[0], c.pr[1], c.pr[2], __longlong_as_double((long long)meta));
#endif
}
// plain (generic-path) value access for the per-stage kernels
struct PVals { double pn; d3 pt, pr; uint32_t meta; };
__device__ __forceinline__ PVals prec_get(const PRec *P, const CRec *rec, int64_t k)
{
    PRaw r;
#if SWEEP_PMODE == 0
    const float *f = reinterpret_cast<const float *>(P + k);
    r.a = make_float4(f[0], f[1], f[2], f[3]);
    r.b = make_float4(f[4], f[5], f[6], f[7]);
#elif SWEEP_PMODE == 1
    r.a = reinterpret_cast<const double4 *>(P)[k];
#else
    r.a = reinterpret_cast<const double4 *>(P)[2 * k];
    r.b = reinterpret_cast<const double4 *>(P)[2 * k + 1];
#endif
    PVals v;
    praw_vals(r, v.pn, v.pt, v.pr);
    v.meta = praw_meta(r, reinterpret_cast<const double4 *>(rec)[k]);
    return v;
}
__device__ __forceinline__ void prec_put(PRec *P, int64_t k, double pn, const d3 pt, const d3 pr, uint32_t meta)
{
    ContactOutT<PN_T, PT_T> c;
    c.pn = (PN_T)pn;
    c.pt[0] = (PT_T)pt.x; c.pt[1] = (PT_T)pt.y; c.pt[2] = (PT_T)pt.z;
    c.pr[0] = (PT_T)pr.x; c.pr[1] = (PT_T)pr.y; c.pr[2] = (PT_T)pr.z;
#if SWEEP_PMODE == 0
    float *f = reinterpret_cast<float *>(P + k);
    f[0] = c.pn; f[1] = c.pt[0]; f[2] = c.pt[1]; f[3] = c.pt[2]; f[4] = c.pr[0]; f[5] = c.pr[1]; f[6] = c.pr[2];
    f[7] = __uint_as_float(meta);
#elif SWEEP_PMODE == 1
    reinterpret_cast<double4 *>(P)[k] = make_double4(c.pn, pk2(c.pt[0], c.pt[1]), pk2(c.pt[2], c.pr[0]), pk2(c.pr[1], c.pr[2]));
#else
    reinterpret_cast<double4 *>(P)[2 * k] = make_double4(c.pn, c.pt[0], c.pt[1], c.pt[2]);
    reinterpret_cast<double4 *>(P)[2 * k + 1] = make_double4(c.pr[0], c.pr[1], c.pr[2], __longlong_as_double((long long)meta));
#endif
}

// ------------------------------------------------------------------ the sweep kernel
// Each warp takes a contiguous range of the tile's particles holding ~1/NWT of its items
// (balanced: the CTA's final barrier does not wait on a warp of coarse particles) and walks
// their items 32 at a time, the next chunk's records in flight while the current one computes.
// Operands are loaded by index straight into their canonical (a, b) slots (no selects):
// intra-tile pairs and boundary contacts from shared memory, cross-tile pairs from global
// (the tile's own particle is L1/L2-resident: the CTA just staged it).
template <bool IMPACT>
__global__ void __launch_bounds__(TT, SWEEP_MINB)
    k_sweep(int64_t N, const double4 *__restrict__ vin, const double4 *__restrict__ win,
            const double *__restrict__ rad, double4 *__restrict__ vout, double4 *__restrict__ wout,
            const uint32_t *__restrict__ istart, const uint32_t *__restrict__ pin, const CRec *__restrict__ rec,
            const PRec *__restrict__ Pin, PRec *__restrict__ Pout, const DevBoundary *__restrict__ bnd, SolveParams sp)
{
    __shared__ double2 sVa[TT], sVb[TT], sWa[TT], sWb[TT];
    __shared__ double sR[TT];
    __shared__ double2 sSig[TT];          // fixed-point scales (linear, angular) of the particle
    __shared__ long long sAcc[6][TT];
    extern __shared__ long long sSlotDyn[];                 // [6][SLOT_CAP] (dynamic: > 48 KB total)
    long long (*sSlot)[SLOT_CAP] = reinterpret_cast<long long (*)[SLOT_CAP]>(sSlotDyn);
    __shared__ uint32_t sI[TT + 1];
    __shared__ uint32_t sIn[TT];
    __shared__ uint8_t sOwn[NWT][32];
    __shared__ int sBad[TT];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * TT;
    const int np = (int)min((int64_t)TT, N - p0);
    for (int q = t; q <= np; q += TT) sI[q] = __ldg(&istart[p0 + q]);
    if (t < np) {
        const double4 v = ld4g(&vin[p0 + t]), o = ld4g(&win[p0 + t]);
        sVa[t] = make_double2(v.x, v.y); sVb[t] = make_double2(v.z, v.w);
        sWa[t] = make_double2(o.x, o.y); sWb[t] = make_double2(o.z, o.w);
        sR[t] = __ldg(&rad[p0 + t]);
        const uint32_t in = __ldg(&pin[p0 + t]);
        sIn[t] = in;
        const uint32_t c = (__ldg(&istart[p0 + t + 1]) - __ldg(&istart[p0 + t])) + (in >> 16);
        sSig[t] = c ? make_double2(pow2(FX_EL + fx_exp(v.w, c)), pow2(FX_EA + fx_exp(o.w, c))) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int f = 0; f < 6; f++) sAcc[f][t] = 0;
    sBad[t] = 0;
    __syncthreads();
    // the warp's particles [pb, pe): first particle whose items start at or after its share
    const uint32_t I0 = sI[0], IT = sI[np] - I0;
    auto first_at = [&](int q) -> int {
        if (q <= 0) return 0;
        if (q >= NWT) return np;
        const uint32_t tgt = I0 + (uint32_t)(((uint64_t)IT * (uint32_t)q + NWT - 1) / NWT);
        int lo = 0, hi = np;                 // smallest p in [0, np] with sI[p] >= tgt
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (sI[mid] < tgt) lo = mid + 1; else hi = mid; }
        return lo;
    };
    const int pb = first_at(w), pe = first_at(w + 1);
    const uint32_t k0 = sI[pb], k1 = sI[pe];
    int carry = 0;
    double4 cn;
    PRaw qn;
    if (k0 + lane < k1) { cn = ldg4d(rec + k0 + lane); qn = ld_praw(Pin, k0 + lane); }
    for (uint32_t kb = k0; kb < k1; kb += 32) {
        const uint32_t k = kb + lane;
        const bool valid = k < k1;
        const double4 cr = cn;
        const PRaw q = qn;
        if (kb + 32 + lane < k1) { cn = ldg4d(rec + kb + 32 + lane); qn = ld_praw(Pin, kb + 32 + lane); }   // next chunk in flight
        // segment starts of the chunk (particles of the warp whose first item lies in it)
        unsigned smask = 0;
        for (int g = pb; g < pe; g += 32) {
            const int p = g + lane;
            const uint32_t sp_ = p < pe ? sI[p] : 0u, ep = p < pe ? sI[p + 1] : 0u;
            const bool st = ep > sp_ && sp_ >= kb && sp_ < kb + 32;
            smask |= __reduce_or_sync(0xffffffffu, st ? (1u << (sp_ - kb)) : 0u);
            if (st) sOwn[w][sp_ - kb] = (uint8_t)p;
        }
        __syncwarp();
        const unsigned le = smask & (0xffffffffu >> (31 - lane));
        const int sstart = le ? 31 - __clz(le) : 0;
        const int o = le ? (int)sOwn[w][sstart] : carry;
        long long v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, v5 = 0;
        if (valid) {
            const uint32_t meta = praw_meta(q, cr);
            const bool intra = (meta & IT_INTRA) != 0, isB = (meta & IT_B) != 0, ext = (meta & IT_EXT) != 0;
            double4 VA, WA, VB, WB;
            double ra, rb, mt, mr;
            int pl = -1;
            if (ext) {           // the particle is body a, the wall / plate body b
                d3 bv;
                boundary_body((meta & IT_IDX) | PARTNER_EXT, bnd, bv, mt, mr);
                VA = cat2(sVa[o], sVb[o]); WA = cat2(sWa[o], sWb[o]); ra = sR[o];
                VB = make_double4(bv.x, bv.y, bv.z, 0.0);
                WB = make_double4(0.0, 0.0, 0.0, 0.0);
                rb = 0.0;
            } else {
                mt = sp.mu_t;
                mr = sp.mu_r;
                if (intra) {     // owned by body a; body b in the tile
                    pl = (int)(meta & IT_LOC);
                    VA = cat2(sVa[o], sVb[o]); WA = cat2(sWa[o], sWb[o]); ra = sR[o];
                    VB = cat2(sVa[pl], sVb[pl]); WB = cat2(sWa[pl], sWb[pl]); rb = sR[pl];
                } else {
                    const int64_t g = (int64_t)(meta & IT_IDX), me = p0 + o;
                    const int64_t ga = isB ? g : me, gb = isB ? me : g;
                    VA = ld4g(&vin[ga]); WA = ld4g(&win[ga]); ra = __ldg(&rad[ga]);
                    VB = ld4g(&vin[gb]); WB = ld4g(&win[gb]); rb = __ldg(&rad[gb]);
                }
            }
            d3 n;
            double delta, bias;
            crec_decode(cr, n, delta, bias);
            const double Rs = ext ? ra : rstar(ra, rb);
            const double S = IMPACT ? 0.0 : spook_sigma(sp, Rs, delta);
            const double la = ra - 0.5 * delta, lb = ext ? 0.0 : rb - 0.5 * delta;
            double Pn0;
            d3 Pt0, Pr0;
            praw_vals(q, Pn0, Pt0, Pr0);
            const ContactOutT<PN_T, PT_T> c = contact_core_t<PN_T, PT_T>(VA, WA, VB, WB, mt, n, mr * Rs, S, bias, la, lb,
                                                                         Pn0, Pt0, Pr0, sp.rolling_dims);
            st_prec(Pout, k, c, meta);
            bool bad = false;
            if (intra) {   // body b of an intra-tile contact: its slot (stored first: fewer live registers)
                const double2 sg = sSig[pl];
                const Fx6 ot = fx6(c.L, share_b(lb, c.nxdPt, c.dPr), sg.x, sg.y, bad);
                const int sl = (int)((meta >> IT_SLOT_SHIFT) & IT_SLOT_MASK);
#pragma unroll
                for (int f = 0; f < 6; f++) sSlot[f][sl] = ot.v[f];
                if (bad) atomicOr(&sBad[pl], 1);
            }
            const double2 ss = sSig[o];
            const d3 Ls = isB ? c.L : mk(-c.L.x, -c.L.y, -c.L.z);
            const d3 As = isB ? share_b(lb, c.nxdPt, c.dPr) : share_a(la, c.nxdPt, c.dPr);
            const Fx6 me6 = fx6(Ls, As, ss.x, ss.y, bad);
            v0 = me6.v[0]; v1 = me6.v[1]; v2 = me6.v[2]; v3 = me6.v[3]; v4 = me6.v[4]; v5 = me6.v[5];
            if (bad) atomicOr(&sBad[o], 1);
        }
        // segmented sum of the self shares (items are grouped by owner): exact int64
        const int dist = valid ? lane - sstart : 0;
        const int maxd = __reduce_max_sync(0xffffffffu, dist);
        for (int d = 1; d <= maxd; d <<= 1) {
            const long long u0 = __shfl_up_sync(0xffffffffu, v0, d), u1 = __shfl_up_sync(0xffffffffu, v1, d);
            const long long u2 = __shfl_up_sync(0xffffffffu, v2, d), u3 = __shfl_up_sync(0xffffffffu, v3, d);
            const long long u4 = __shfl_up_sync(0xffffffffu, v4, d), u5 = __shfl_up_sync(0xffffffffu, v5, d);
            if (lane - d >= sstart) {     // mod 2^64 (raw patterns)
                v0 = (long long)((unsigned long long)v0 + (unsigned long long)u0);
                v1 = (long long)((unsigned long long)v1 + (unsigned long long)u1);
                v2 = (long long)((unsigned long long)v2 + (unsigned long long)u2);
                v3 = (long long)((unsigned long long)v3 + (unsigned long long)u3);
                v4 = (long long)((unsigned long long)v4 + (unsigned long long)u4);
                v5 = (long long)((unsigned long long)v5 + (unsigned long long)u5);
            }
        }
        const bool seg_end = valid && (lane == 31 || ((smask >> (lane + 1)) & 1u) || k + 1 >= k1);
        if (seg_end) {
            unsigned long long *A0 = reinterpret_cast<unsigned long long *>(&sAcc[0][0]);
            A0[0 * TT + o] += (unsigned long long)v0; A0[1 * TT + o] += (unsigned long long)v1;
            A0[2 * TT + o] += (unsigned long long)v2; A0[3 * TT + o] += (unsigned long long)v3;
            A0[4 * TT + o] += (unsigned long long)v4; A0[5 * TT + o] += (unsigned long long)v5;
        }
        carry = __shfl_sync(0xffffffffu, o, 31);
        __syncwarp();
    }
    __syncthreads();
    if (t < np) {
        double4 V = cat2(sVa[t], sVb[t]), W = cat2(sWa[t], sWb[t]);
        const uint32_t in = sIn[t], is = in & 0xFFFFu, ic = in >> 16;
        const uint32_t cnt = (sI[t + 1] - sI[t]) + ic;      // contacts of the particle (mass splitting)
        if (cnt) {
            long long a[6];
#pragma unroll
            for (int f = 0; f < 6; f++) a[f] = sAcc[f][t];
            for (uint32_t s = is; s < is + ic; s++) {
#pragma unroll
                for (int f = 0; f < 6; f++) a[f] = (long long)((unsigned long long)a[f] + (unsigned long long)sSlot[f][s]);
            }
            const unsigned long long mc = (unsigned long long)cnt * (unsigned long long)FX_MAGIC_BITS;
#pragma unroll
            for (int f = 0; f < 6; f++) a[f] = (long long)((unsigned long long)a[f] - mc);
            // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
            const double2 sg = sSig[t];
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            const double qL = (1.0 / sg.x) * im, qA = (1.0 / sg.y) * iI;   // 1/s exact (powers of two)
            V.x += (double)a[0] * qL; V.y += (double)a[1] * qL; V.z += (double)a[2] * qL;
            W.x += (double)a[3] * qA; W.y += (double)a[4] * qA; W.z += (double)a[5] * qA;
            if (sBad[t]) { V.x = __longlong_as_double(0x7FF8000000000000LL); }
        }
        st4g(&vout[p0 + t], V);
        st4g(&wout[p0 + t], W);
    }
}

void launch_sweep_items(bool impact, int64_t N, const double4 *vin, const double4 *win, const double *rad, double4 *vout,
                        double4 *wout, const SweepPlan &pl, const CRec *rec, const PRec *Pin, PRec *Pout,
                        const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    constexpr int dyn = 6 * SLOT_CAP * (int)sizeof(long long);
    static bool attr = [] {
        cudaFuncSetAttribute(k_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        cudaFuncSetAttribute(k_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        return true;
    }();
    (void)attr;
    const unsigned gb = (unsigned)((N + TT - 1) / TT);
    if (impact)
        k_sweep<true><<<gb, TT, dyn, s>>>(N, vin, win, rad, vout, wout, pl.istart, pl.pin, rec, Pin, Pout, bnd, sp);
    else
        k_sweep<false><<<gb, TT, dyn, s>>>(N, vin, win, rad, vout, wout, pl.istart, pl.pin, rec, Pin, Pout, bnd, sp);
}

// ================================================================== the tile plan (per step)
// Particle i's half-contacts (incidence CSR) split into its items and its incoming slots.
__device__ __forceinline__ bool half_is_intra(uint2 ent, int64_t i, const uint8_t *noint)
{
    if (ent.y & PARTNER_EXT) return false;
    const int64_t ti = i / TT;
    return (int64_t)ent.y / TT == ti && !noint[ti];
}

// counts per particle: items (owned halves) and incoming slots (body b of an intra contact)
__global__ void k_plan_count(int64_t N, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                             const uint8_t *__restrict__ noint, uint32_t *__restrict__ nitem, uint32_t *__restrict__ nin)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    uint32_t a = 0, b = 0;
    for (uint32_t k = inc_start[i]; k < inc_start[i + 1]; k++) {
        const uint2 e = inc[k];
        if ((e.x & B_SIDE) && half_is_intra(e, i, noint)) b++;
        else a++;
    }
    nitem[i] = a;
    nin[i] = b;
}

// per tile: slot offsets of its particles (block scan); a tile whose intra contacts exceed the
// slot capacity evaluates them all as cross pairs instead (flag, recounted by the caller)
__global__ void __launch_bounds__(TT) k_plan_tile(int64_t N, const uint32_t *__restrict__ nin, uint32_t *__restrict__ pin,
                                                  uint8_t *__restrict__ noint, unsigned int *__restrict__ any_full)
{
    __shared__ uint32_t sw[NWT];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t i = (int64_t)blockIdx.x * TT + t;
    const uint32_t x = i < N ? nin[i] : 0u;
    uint32_t inc = x;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += u;
    }
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    uint32_t base = 0, tot = 0;
    for (int q = 0; q < NWT; q++) { if (q < w) base += sw[q]; tot += sw[q]; }
    const bool full = tot > (uint32_t)SLOT_CAP;
    if (i < N) pin[i] = full ? 0u : ((base + inc - x) | (x << 16));
    if (t == 0) {
        noint[blockIdx.x] = full ? 1 : 0;
        if (full) atomicOr(any_full, 1u);
    }
}

// slot of each intra contact at its body b
__global__ void k_plan_slot(int64_t N, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                            const uint8_t *__restrict__ noint, const uint32_t *__restrict__ pin,
                            uint32_t *__restrict__ slot_of)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    uint32_t s = pin[i] & 0xFFFFu;
    for (uint32_t k = inc_start[i]; k < inc_start[i + 1]; k++) {
        const uint2 e = inc[k];
        if ((e.x & B_SIDE) && half_is_intra(e, i, noint)) slot_of[e.x & INC_CMASK] = s++;
    }
}

// items of particle i at istart[i]: contact index and meta word
__global__ void k_plan_fill(int64_t N, const uint32_t *__restrict__ inc_start, const uint2 *__restrict__ inc,
                            const uint8_t *__restrict__ noint, const uint32_t *__restrict__ istart,
                            const uint32_t *__restrict__ slot_of, uint32_t *__restrict__ item_c,
                            uint32_t *__restrict__ item_meta)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    uint32_t o = istart[i];
    const int64_t tb = (i / TT) * TT;
    for (uint32_t k = inc_start[i]; k < inc_start[i + 1]; k++) {
        const uint2 e = inc[k];
        const uint32_t c = e.x & INC_CMASK;
        const bool isB = (e.x & B_SIDE) != 0;
        const bool intra = half_is_intra(e, i, noint);
        if (isB && intra) continue;
        uint32_t meta;
        if (e.y & PARTNER_EXT) meta = IT_EXT | (e.y & ~PARTNER_EXT);
        else if (intra) meta = IT_INTRA | (uint32_t)((int64_t)e.y - tb) | (slot_of[c] << IT_SLOT_SHIFT);
        else meta = (isB ? IT_B : 0u) | e.y;
        item_c[o] = c;
        item_meta[o] = meta;
        o++;
    }
}

// per particle radius (read by the sweeps: lever arms, R*)
__global__ void k_radius(int64_t N, const double4 *__restrict__ pos, double *__restrict__ rad)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) rad[i] = pos[i].w;
}

#define IGRID(n) (unsigned)(((n) + 255) / 256), 256, 0, s
// Builds pl for this step's incidence; returns the item count through *nitems (host sync).
// Scratch: nitem (N+1), nin (N) u32; pl arrays sized by the caller (istart N+1, pin N, noint
// ceil(N/TT), slot_of nc).  Items must then be filled with plan_fill once *nitems is sized.
void plan_counts(int64_t N, const uint32_t *inc_start, const uint2 *inc, const SweepPlan &pl, uint32_t *nitem,
                 uint32_t *nin, unsigned int *any_full, void *scan_tmp, cudaStream_t s, long long *launches)
{
    const int64_t nt = (N + TT - 1) / TT;
    cudaMemsetAsync(pl.noint, 0, nt ? nt : 1, s);
    cudaMemsetAsync(any_full, 0, sizeof(unsigned int), s);
    if (N) {
        k_plan_count<<<IGRID(N)>>>(N, inc_start, inc, pl.noint, nitem, nin);
        k_plan_tile<<<(unsigned)nt, TT, 0, s>>>(N, nin, pl.pin, pl.noint, any_full);
        // tiles over capacity: recount with their intra pairs as cross pairs
        k_plan_count<<<IGRID(N)>>>(N, inc_start, inc, pl.noint, nitem, nin);
        k_plan_slot<<<IGRID(N)>>>(N, inc_start, inc, pl.noint, pl.pin, pl.slot_of);
    }
    scan_u32(nitem, pl.istart, N, scan_tmp, s, launches);
    *launches += N ? 4 : 0;
}
void plan_fill(int64_t N, const uint32_t *inc_start, const uint2 *inc, const double4 *pos, const SweepPlan &pl,
               cudaStream_t s, long long *launches)
{
    if (!N) return;
    k_plan_fill<<<IGRID(N)>>>(N, inc_start, inc, pl.noint, pl.istart, pl.slot_of, pl.item_c, pl.item_meta);
    k_radius<<<IGRID(N)>>>(N, pos, pl.rad);
    *launches += 2;
}

// ------------------------------------------------------------------ per stage: records in, impulses out
__global__ void k_item_pack(int64_t n, const uint32_t *__restrict__ item_c, const uint32_t *__restrict__ item_meta,
                            const G4 *__restrict__ geo, const double *__restrict__ cdel, const R4 *__restrict__ row,
                            const P4 *__restrict__ Pa, const P4 *__restrict__ Pb, CRec *__restrict__ rec,
                            PRec *__restrict__ P)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t c = item_c[k], meta = item_meta[k];
    const G4 g = geo[c];
    reinterpret_cast<double4 *>(rec)[k] = crec_encode(mk(g.x, g.y, g.z), cdel[c], row[c].y, meta);
    if (Pa) {
        const P4 a = Pa[c], b = Pb[c];
        prec_put(P, k, a.x, mk(a.y, a.z, a.w), mk(b.x, b.y, b.z), meta);
    } else {
        prec_put(P, k, 0.0, mk(0, 0, 0), mk(0, 0, 0), meta);
    }
}
// the stage's final impulses back to the contact arrays (one item per contact writes: body a's)
__global__ void k_item_unpack(int64_t n, const uint32_t *__restrict__ item_c, const CRec *__restrict__ rec,
                              const PRec *__restrict__ P, P4 *__restrict__ Pa, P4 *__restrict__ Pb)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const PVals q = prec_get(P, rec, k);
    if (q.meta & IT_B) return;
    const uint32_t c = item_c[k];
    Pa[c] = make_float4((float)q.pn, (float)q.pt.x, (float)q.pt.y, (float)q.pt.z);
    Pb[c] = make_float4((float)q.pr.x, (float)q.pr.y, (float)q.pr.z, 0.0f);
}
void item_pack(int64_t n, const SweepPlan &pl, const G4 *geo, const double *cdel, const R4 *row, const P4 *Pa,
               const P4 *Pb, CRec *rec, PRec *P, cudaStream_t s)
{ if (n) k_item_pack<<<IGRID(n)>>>(n, pl.item_c, pl.item_meta, geo, cdel, row, Pa, Pb, rec, P); }
void item_unpack(int64_t n, const SweepPlan &pl, const CRec *rec, const PRec *P, P4 *Pa, P4 *Pb, cudaStream_t s)
{ if (n) k_item_unpack<<<IGRID(n)>>>(n, pl.item_c, rec, P, Pa, Pb); }

// ------------------------------------------------------------------ monolithic plates (R18b)
// owned plate items of the step
__global__ void k_plate_items_flag(int64_t n, const uint8_t *__restrict__ own, const uint32_t *__restrict__ item_c,
                                   const uint32_t *__restrict__ item_meta, const uint2 *__restrict__ cij,
                                   uint32_t *__restrict__ flag)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t m = item_meta[k];
    flag[k] = ((m & IT_EXT) && (m & PARTNER_PLATE) && (!own || own[cij[item_c[k]].x])) ? 1u : 0u;
}
void launch_plate_items_flag(int64_t n, const uint8_t *own, const SweepPlan &pl, const uint2 *cij, uint32_t *flag,
                             cudaStream_t s)
{ if (n) k_plate_items_flag<<<IGRID(n)>>>(n, own, pl.item_c, pl.item_meta, cij, flag); }
// the impulse a plate received over a sweep from its items (in == nullptr: all of out)
__global__ void k_plate_hub_items(int64_t n, const uint32_t *__restrict__ list, const uint32_t *__restrict__ item_c,
                                  const uint32_t *__restrict__ item_meta, const G4 *__restrict__ geo,
                                  const CRec *__restrict__ rec, const PRec *__restrict__ pin,
                                  const PRec *__restrict__ pout, unsigned long long *__restrict__ acc)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t k = list[t];
    const PVals o = prec_get(pout, rec, k);
    const int q = (item_meta[k] >> 4) & 0xF;
    const G4 g = geo[item_c[k]];
    double i0 = 0;
    d3 it = mk(0, 0, 0);
    if (pin) { const PVals i = prec_get(pin, rec, k); i0 = i.pn; it = i.pt; }
    const double dPn = o.pn - i0;
    const double d[3] = {dPn * g.x + (o.pt.x - it.x), dPn * g.y + (o.pt.y - it.y), dPn * g.z + (o.pt.z - it.z)};
    for (int k2 = 0; k2 < 3; k2++) atomicAdd(&acc[3 * q + k2], (unsigned long long)llrint(d[k2] * HUB_SCALE));
}
void launch_plate_hub_items(int64_t n, const uint32_t *list, const SweepPlan &pl, const G4 *geo, const CRec *rec,
                            const PRec *pin, const PRec *pout, unsigned long long *acc, cudaStream_t s)
{ if (n) k_plate_hub_items<<<IGRID(n)>>>(n, list, pl.item_c, pl.item_meta, geo, rec, pin, pout, acc); }
#undef IGRID
