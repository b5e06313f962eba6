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
// A tile's items are stored contiguously, grouped by owner (each warp takes a range of whole
// particles, plan k_plan_warps), so records move with coalesced 256-bit accesses; the tile's
// particle states land in shared memory by TMA bulk copies on an mbarrier:
//   CRec 32 B per item: n (a -> b) and delta, fp64 (the item's meta word in n's low bits)
//   PRec 64 B per item: P_n, P_t (3), P_r (3) and the stage's SPOOK bias b, fp64
// Everything else the contact row needs is derived from the radii: R* = r_a r_b/(r_a + r_b),
// l_a = r_a - delta/2, l_b = r_b - delta/2, mu_r R*, Sigma-hat = Cs / sqrt(2 R* delta) (R4).
//
// Reduction (deterministic, decomposition-invariant, no float atomics).  Each body's share of a
// contact increment is converted to int64 fixed point with a power-of-two scale chosen from the
// body's own mass-splitting weight (c/m, c/I) and summed exactly; integer sums are order-free,
// so a particle's velocity update does not depend on how contacts fall into tiles, warps or
// ranks: trajectories are bit-identical for any decomposition.  Resolution
// ~2^-42 m/s (linear) and ~2^-36 rad/s (angular) of velocity per contribution (5e-9 of g dt,
// against 1e-5 of the parity bar); a contribution beyond 2^51 units (~500 m/s or ~3e4 rad/s in
// one sweep) or a non-finite one poisons the particle's velocity with NaN (the step rolls back,
// S:385).
#include "common.cuh"
#include "kernels.h"
#include "sweep_core.cuh"

constexpr int TT = SWEEP_TILE;           // particles per tile (one CTA), kernels.h
constexpr int NWT = TT / 32;
constexpr int SLOT_CAP = SWEEP_SLOT_CAP; // intra-tile body-b slots per tile
static_assert(TT % 32 == 0 && TT <= 512, "tile: whole warps, owner index in 9 bits");
static_assert(SLOT_CAP <= (int)IT_SLOT_MASK + 1 && SLOT_CAP < 65536, "slot index: 12 bits in the meta word");
constexpr int FX_EL = 42, FX_EA = 36;    // fixed-point exponents (linear, angular)

// DEM_CHECK builds (tests only, never shipped): index invariants of the tile plan trap
#ifdef DEM_CHECK
#define SW_CHECK(c, what)                                                                          \
    do {                                                                                           \
        if (!(c)) {                                                                                \
            printf("k_sweep check failed: %s (tile %lld thread %d)\n", what, (long long)blockIdx.x, \
                   (int)threadIdx.x);                                                              \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define SW_CHECK(c, what) ((void)0)
#endif

__device__ __forceinline__ double4 cat2(const double2 a, const double2 b) { return make_double4(a.x, a.y, b.x, b.y); }

// ------------------------------------------------------------------ fixed point
// Scale of body i: 2^(E + ilogb(w_i) - floor(log2 c_i)) ~ 2^E m_i (w = c/m, c = contact count;
// likewise with c/I): integer units of 2^-E m/s (rad/s) of velocity, whatever the particle size.
__device__ __forceinline__ int fx_exp(double w, uint32_t c)
{
    return (int)((__double_as_longlong(w) >> 52) & 0x7FF) - 1023 - (31 - __clz((int)c));
}
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }
// the (linear, angular) scales from their exponents packed as two int16 (SWEEP_SIG16)
__device__ __forceinline__ double2 sig2(int x) { return make_double2(pow2((int)(short)(x & 0xFFFF)), pow2(x >> 16)); }
// Fixed-point value of x s (s a power of two, so x s is exact), kept as raw bits: t = x s + 1.5 2^52
// rounds x s to an integer exactly (RN-even, like llrint) whenever |x s| <= 2^51, and then the
// bit pattern of t is round(x s) + FX_MAGIC_BITS.  Sums of raw patterns are taken mod 2^64 and
// the c FX_MAGIC_BITS are subtracted once per particle (exact: integer arithmetic wraps).  fx1
// returns the deviation of t's exponent field from 0x433: nonzero means out of range or NaN.
constexpr double FX_MAGIC = 6755399441055744.0;            // 1.5 2^52
constexpr long long FX_MAGIC_BITS = 0x4338000000000000LL;
struct Fx6 { long long v[6]; };
__device__ __forceinline__ unsigned fx1(double x, double s, long long &o)
{
    o = __double_as_longlong(__fma_rn(x, s, FX_MAGIC));
    return ((unsigned)((unsigned long long)o >> 52)) ^ 0x433u;
}
__device__ __forceinline__ Fx6 fx6(const d3 L, const d3 A, double sL, double sA, bool &bad)
{
    Fx6 o;
    const unsigned e = fx1(L.x, sL, o.v[0]) | fx1(L.y, sL, o.v[1]) | fx1(L.z, sL, o.v[2]) | fx1(A.x, sA, o.v[3]) |
                       fx1(A.y, sA, o.v[4]) | fx1(A.z, sA, o.v[5]);
    bad |= e != 0u;
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

// ------------------------------------------------------------------ item records
// CRec (32 B, written per stage): n (a -> b) and delta in fp64; the item's 32-bit meta word
// rides in the low 16 bits of n.x and n.y (n keeps 36 mantissa bits there: ~1e-11), the owner's
// index in the tile in the low 9 bits of delta (43 bits left: ~1e-13).
// PRec (64 B, ping-pong): P_n, P_t (3), P_r (3) and the stage's SPOOK bias b, all fp64.  fp64
// impulses are what the 1e-5 force/torque bar needs: with fp32 storage the rounding of the
// impulses at every sweep, amplified by the rigid friction and rolling rows, reaches 6.8e-5 in
// torque on the bench-shaped bed (measured); fp64 storage gives 9e-8.
constexpr unsigned long long N_LOWMASK = 0xFFFFull;
__device__ __forceinline__ double clr_low(double x)
{
    return __longlong_as_double((long long)((unsigned long long)__double_as_longlong(x) & ~N_LOWMASK));
}
__device__ __forceinline__ uint32_t crec_meta(const double4 c)
{
    return (uint32_t)((unsigned long long)__double_as_longlong(c.x) & N_LOWMASK) |
           ((uint32_t)((unsigned long long)__double_as_longlong(c.y) & N_LOWMASK) << 16);
}
constexpr unsigned long long OWN_MASK = 0x1FFull;    // owner index bits in delta (tiles <= 512)
__device__ __forceinline__ int crec_owner(const double4 c) { return (int)((unsigned long long)__double_as_longlong(c.w) & OWN_MASK); }
__device__ __forceinline__ double crec_delta(const double4 c)
{
    return __longlong_as_double((long long)((unsigned long long)__double_as_longlong(c.w) & ~OWN_MASK));
}
__device__ __forceinline__ double4 crec_encode(const d3 n, double delta, uint32_t meta, uint32_t owner)
{
    const double nx = __longlong_as_double((long long)(((unsigned long long)__double_as_longlong(n.x) & ~N_LOWMASK) |
                                                       (meta & 0xFFFFu)));
    const double ny = __longlong_as_double((long long)(((unsigned long long)__double_as_longlong(n.y) & ~N_LOWMASK) |
                                                       (meta >> 16)));
    const double dl = __longlong_as_double((long long)(((unsigned long long)__double_as_longlong(delta) & ~OWN_MASK) | owner));
    return make_double4(nx, ny, n.z, dl);
}
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
struct PRaw { double4 a, b; };       // (P_n, P_t) and (P_r, bias)
__device__ __forceinline__ PRaw ld_praw(const PRec *P, uint32_t k)
{
    PRaw r;
    r.a = ldg4d(P + k);
    r.b = ldg4d(reinterpret_cast<const double4 *>(P + k) + 1);
    return r;
}

// ------------------------------------------------------------------ the sweep kernel
// One CTA per tile of TT consecutive particles (2 CTAs per SM).  The tile's particle states are
// staged into shared memory with cp.async.  Each warp takes a contiguous range of the tile's
// particles holding ~1/NWT of its items (plan k_plan_warps: the tile's final barrier does not
// wait on a warp of coarse particles) and walks their items 32 at a time, the next chunk's item
// records in flight (registers) while the current chunk computes.  Operands are loaded by index
// straight into their canonical (a, b) slots (no selects): the tile's particles from shared
// memory, the partner of a cross-tile pair from global memory.
// Measured and dropped (profiles/r02_sweep_variants.jsonl): the next chunk's cross-tile partners
// gathered by cp.async into a shared-memory ring (3.55 ms vs 3.03) or prefetched into L1 (3.24),
// warps taking the tile's chunks round robin with smem atomics at chunk edges (3.17).
__device__ __forceinline__ void cp_async16(void *s, const void *g)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void *s, const void *g)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(void *s, const void *g)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

#if SWEEP_TMA
// the tile's particle states as in HBM (double4 v, w), radii, item starts and incoming-slot
// words, each landed by one TMA bulk copy (cp.async.bulk) on an mbarrier: no per-thread copies
struct StageBuf {
    double4 v[TT], w[TT];
    double r[TT];
    uint32_t is[TT + 4];
    uint32_t in[TT];
};
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t up16(uint32_t b) { return (b + 15u) & ~15u; }
// one thread: arm the barrier with the byte count and issue the five copies (sizes rounded up to
// 16 B; the plan arrays and radii carry the padding, ctx.cu alloc_particles)
__device__ __forceinline__ void stage_tile_tma(StageBuf &B, uint64_t *bar, int64_t p0, int np, const double4 *vin,
                                               const double4 *win, const double *rad, const uint32_t *istart,
                                               const uint32_t *pin)
{
    const uint32_t bv = (uint32_t)np * 32u, br = up16((uint32_t)np * 8u), bi = up16((uint32_t)(np + 1) * 4u),
                   bn = up16((uint32_t)np * 4u);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(2 * bv + br + bi + bn)
                 : "memory");
    bulk_g2s(B.v, vin + p0, bv, bar);
    bulk_g2s(B.w, win + p0, bv, bar);
    bulk_g2s(B.r, rad + p0, br, bar);
    bulk_g2s(B.is, istart + p0, bi, bar);
    bulk_g2s(B.in, pin + p0, bn, bar);
}
__device__ __forceinline__ void mbar_wait0(uint64_t *bar)
{
    asm volatile("{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT%=;\n}"
                 ::"r"(smem_u32(bar)) : "memory");
}
#define SV(i) (B.v[i])
#define SW(i) (B.w[i])
#else
// the tile's particle states (v and w as double2 halves: conflict-free 16-byte reads), radii,
// item starts and incoming-slot words
struct StageBuf {
    double2 va[TT], vb[TT], wa[TT], wb[TT];
    double r[TT];
    uint32_t is[TT + 1];
    uint32_t in[TT];
};
__device__ __forceinline__ void stage_tile(StageBuf &B, int64_t p0, int np, int t, const double4 *vin,
                                           const double4 *win, const double *rad, const uint32_t *istart,
                                           const uint32_t *pin)
{
    // 16-byte chunk c of the tile's v (w) array: particle c/2, half c%2; consecutive threads take
    // consecutive chunks, so a warp reads 512 contiguous bytes and writes two 256-byte runs
    const double2 *v = reinterpret_cast<const double2 *>(vin + p0), *o = reinterpret_cast<const double2 *>(win + p0);
    for (int c = t; c < 2 * np; c += TT) {
        double2 *dv = (c & 1) ? B.vb : B.va, *dw = (c & 1) ? B.wb : B.wa;
        cp_async16(&dv[c >> 1], v + c);
        cp_async16(&dw[c >> 1], o + c);
    }
    if (t < np) {
        cp_async8(&B.r[t], rad + p0 + t);
        cp_async4(&B.in[t], pin + p0 + t);
    }
    for (int q = t; q <= np; q += TT) cp_async4(&B.is[q], istart + p0 + q);
    cp_async_commit();
}
#define SV(i) cat2(B.va[i], B.vb[i])
#define SW(i) cat2(B.wa[i], B.wb[i])
#endif

template <bool IMPACT>
__global__ void __launch_bounds__(TT, SWEEP_MINB)
    k_sweep(int64_t N, const double4 *__restrict__ vin, const double4 *__restrict__ win,
            const double *__restrict__ rad, double4 *__restrict__ vout, double4 *__restrict__ wout,
            const uint32_t *__restrict__ istart, const uint32_t *__restrict__ pin, const CRec *__restrict__ rec,
            const PRec *__restrict__ Pin, PRec *__restrict__ Pout, const DevBoundary *__restrict__ bnd,
            const uint32_t *__restrict__ wrange, SolveParams sp)
{
    // dynamic shared memory (> 48 KB in total): the tile's states and the body-b slots
    extern __shared__ double2 sDyn[];
    StageBuf &B = *reinterpret_cast<StageBuf *>(sDyn);
    longlong2 *sSlot = reinterpret_cast<longlong2 *>(&B + 1);   // [SLOT_CAP][3]
#if SWEEP_SIG16
    __shared__ int sSig[TT];              // fixed-point scale exponents (linear: low int16, angular: high)
    __shared__ long long sAcc[6][TT];
    __shared__ unsigned sBad[NWT];        // one bit per particle: a share out of range (poisons it)
#define SIG(i) sig2(sSig[i])
#define BAD_SET(i) atomicOr(&sBad[(i) >> 5], 1u << ((i) & 31))
#define BAD_GET(i) ((sBad[(i) >> 5] >> ((i) & 31)) & 1u)
#else
    __shared__ double2 sSig[TT];          // fixed-point scales (linear, angular) of the particle
    __shared__ long long sAcc[6][TT];
    __shared__ int sBad[TT];
#define SIG(i) sSig[i]
#define BAD_SET(i) atomicOr(&sBad[i], 1)
#define BAD_GET(i) sBad[i]
#endif
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t tile = blockIdx.x;
    const int64_t p0 = tile * TT;
    const int np = (int)min((int64_t)TT, N - p0);
#if SWEEP_TMA
    __shared__ __align__(8) uint64_t sBar;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sBar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_tile_tma(B, &sBar, p0, np, vin, win, rad, istart, pin);
    }
#else
    stage_tile(B, p0, np, t, vin, win, rad, istart, pin);
#endif
    // the warp's items [k0, k1) and its first chunk's records, requested before the wait
    const uint32_t k0 = __ldg(&wrange[(size_t)tile * (NWT + 1) + w]), k1 = __ldg(&wrange[(size_t)tile * (NWT + 1) + w + 1]);
    double4 cn;
    PRaw qn;
    if (k0 + lane < k1) { cn = ldg4d(rec + k0 + lane); qn = ld_praw(Pin, k0 + lane); }
#if SWEEP_TMA
    __syncthreads();                      // the barrier is initialised
    mbar_wait0(&sBar);                    // the tile's states are in shared memory
#else
    cp_async_wait_all();
    __syncthreads();                      // the tile's states are in shared memory
#endif
    const double *sR = B.r;
    if (t < np) {
        const uint32_t c = (B.is[t + 1] - B.is[t]) + (B.in[t] >> 16);
#if SWEEP_SIG16
        sSig[t] = c ? (((FX_EL + fx_exp(SV(t).w, c)) & 0xFFFF) | ((FX_EA + fx_exp(SW(t).w, c)) << 16)) : 0;
#else
        sSig[t] = c ? make_double2(pow2(FX_EL + fx_exp(SV(t).w, c)), pow2(FX_EA + fx_exp(SW(t).w, c)))
                    : make_double2(0.0, 0.0);
#endif
    }
#pragma unroll
    for (int f = 0; f < 6; f++) sAcc[f][t] = 0;
#if SWEEP_SIG16
    if (t < NWT) sBad[t] = 0u;
#else
    sBad[t] = 0;
#endif
    __syncthreads();
    // one chunk of 32 items from records (cr, q).  (Unrolling the loop twice, so that the next
    // chunk's records land in a second register set without copies, measured slower: 3.00 ms vs
    // 2.80, profiles/r02_sweep_variants.jsonl.)
    auto chunk = [&](const uint32_t kb, const double4 &cr, const PRaw &q) {
        const uint32_t k = kb + lane;
        const bool valid = k < k1;
        // segments of the chunk: runs of equal owner (items are grouped by owner)
        const int o = valid ? crec_owner(cr) : -1;
        SW_CHECK(!valid || o < np, "owner inside the tile");
        const int op = __shfl_up_sync(0xffffffffu, o, 1);
        const unsigned smask = __ballot_sync(0xffffffffu, valid && (lane == 0 || op != o));
        const unsigned le = smask & (0xffffffffu >> (31 - lane));
        const int sstart = le ? 31 - __clz(le) : 0;
        long long v0 = 0, v1 = 0, v2 = 0, v3 = 0, v4 = 0, v5 = 0;
        if (valid) {
            const uint32_t meta = crec_meta(cr);
            const uint32_t kind = meta & (IT_INTRA | IT_EXT);
            const bool intra = kind == IT_INTRA, ext = kind == IT_EXT, isB = (meta & IT_B) != 0;
            double4 VA, WA, VB, WB;
            double ra, rb, mt, mr;
            int pl = -1;
            if (ext) {           // the particle is body a, the wall / plate body b
                d3 bv;
                boundary_body((meta & IT_IDX) | PARTNER_EXT, bnd, bv, mt, mr);
                VA = SV(o); WA = SW(o); ra = sR[o];
                VB = make_double4(bv.x, bv.y, bv.z, 0.0);
                WB = make_double4(0.0, 0.0, 0.0, 0.0);
                rb = 0.0;
            } else {
                mt = sp.mu_t;
                mr = sp.mu_r;
                int ia = -1, ib = -1;      // shared-memory slots of bodies a and b
                int64_t g = -1;
                if (intra) { pl = (int)(meta & IT_LOC); ia = o; ib = pl; SW_CHECK(pl < np && pl != o, "intra partner"); }
                else {
                    g = (int64_t)(meta & IT_IDX);
                    SW_CHECK(g < N && g != p0 + o, "cross partner index");
                    const int64_t l = g - p0;
                    if (l >= 0 && l < np) { ia = isB ? (int)l : o; ib = isB ? o : (int)l; g = -1; }
                }
                if (g < 0) {
                    VA = SV(ia); WA = SW(ia); ra = sR[ia];
                    VB = SV(ib); WB = SW(ib); rb = sR[ib];
                } else {         // cross-tile partner: from global memory
                    // the own particle from the staged tile, placed by select (the TMA staging
                    // does not allocate in L1, so a global re-read would go to L2)
                    const double4 VP = ld4g(&vin[g]), WP = ld4g(&win[g]);
                    const double rp = __ldg(&rad[g]);
                    const double4 VO = SV(o), WO = SW(o);
                    const double ro = sR[o];
                    VA = isB ? VP : VO; WA = isB ? WP : WO; ra = isB ? rp : ro;
                    VB = isB ? VO : VP; WB = isB ? WO : WP; rb = isB ? ro : rp;
                }
            }
            const d3 n = mk(clr_low(cr.x), clr_low(cr.y), cr.z);
            const double delta = crec_delta(cr), bias = q.b.w;
            const double Rs = ext ? ra : rstar(ra, rb);
            const double S = IMPACT ? 0.0 : (sp.hertz ? sp.Cs * rsqrt64_1(2.0 * Rs * delta) : sp.Cs);   // R4
            const double la = ra - 0.5 * delta, lb = ext ? 0.0 : rb - 0.5 * delta;
            const ContactOutT<double, double> c = contact_core_t<double, double>(
                VA, WA, VB, WB, mt, n, mr * Rs, S, bias, la, lb, q.a.x, mk(q.a.y, q.a.z, q.a.w), mk(q.b.x, q.b.y, q.b.z),
                sp.rolling_dims);
            double *po = reinterpret_cast<double *>(Pout + k);
            stg4d(po, c.pn, c.pt[0], c.pt[1], c.pt[2]);
            stg4d(po + 4, c.pr[0], c.pr[1], c.pr[2], bias);
            // shares: body a gets -(L), -(la n x dPt + dPr); body b gets +L, -lb n x dPt + dPr
            bool bad = false;
            if (intra) {   // body b of an intra-tile contact: its slot (stored first: fewer live registers)
                const double2 sg = SIG(pl);
                const Fx6 ot = fx6(c.L, share_b(lb, c.nxdPt, c.dPr), sg.x, sg.y, bad);
                const int sl = (int)((meta >> IT_SLOT_SHIFT) & IT_SLOT_MASK);
                SW_CHECK(sl < SLOT_CAP, "slot capacity");
                sSlot[3 * sl] = make_longlong2(ot.v[0], ot.v[1]);
                sSlot[3 * sl + 1] = make_longlong2(ot.v[2], ot.v[3]);
                sSlot[3 * sl + 2] = make_longlong2(ot.v[4], ot.v[5]);
                if (bad) BAD_SET(pl);
            }
            const double2 ss = SIG(o);
            const d3 Ls = isB ? c.L : mk(-c.L.x, -c.L.y, -c.L.z);
            const d3 As = isB ? share_b(lb, c.nxdPt, c.dPr) : share_a(la, c.nxdPt, c.dPr);
            const Fx6 me6 = fx6(Ls, As, ss.x, ss.y, bad);
            v0 = me6.v[0]; v1 = me6.v[1]; v2 = me6.v[2]; v3 = me6.v[3]; v4 = me6.v[4]; v5 = me6.v[5];
            if (bad) BAD_SET(o);
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
    };
    for (uint32_t kb = k0; kb < k1; kb += 32) {
        const double4 cr = cn;
        const PRaw q = qn;
        if (kb + 32 + lane < k1) { cn = ldg4d(rec + kb + 32 + lane); qn = ld_praw(Pin, kb + 32 + lane); }   // next chunk in flight
        chunk(kb, cr, q);
    }
    __syncthreads();
    if (t < np) {
        double4 V = SV(t), W = SW(t);
        const uint32_t in = B.in[t], is = in & 0xFFFFu, ic = in >> 16;
        const uint32_t cnt = (B.is[t + 1] - B.is[t]) + ic;      // contacts of the particle (mass splitting)
        if (cnt) {
            long long a[6];
#pragma unroll
            for (int f = 0; f < 6; f++) a[f] = sAcc[f][t];
            SW_CHECK(is + ic <= (uint32_t)SLOT_CAP, "incoming slots");
            for (uint32_t s = is; s < is + ic; s++) {
                const longlong2 x0 = sSlot[3 * s], x1 = sSlot[3 * s + 1], x2 = sSlot[3 * s + 2];
                const long long x[6] = {x0.x, x0.y, x1.x, x1.y, x2.x, x2.y};
#pragma unroll
                for (int f = 0; f < 6; f++) a[f] = (long long)((unsigned long long)a[f] + (unsigned long long)x[f]);
            }
            const unsigned long long mc = (unsigned long long)cnt * (unsigned long long)FX_MAGIC_BITS;
#pragma unroll
            for (int f = 0; f < 6; f++) a[f] = (long long)((unsigned long long)a[f] - mc);
            // body update with the real masses (1/m = (c/m)/c): the mass-splitting average
            const double2 sg = SIG(t);
            const double im = V.w / (double)cnt, iI = W.w / (double)cnt;
            const double qL = (1.0 / sg.x) * im, qA = (1.0 / sg.y) * iI;   // 1/s exact (powers of two)
            V.x += (double)a[0] * qL; V.y += (double)a[1] * qL; V.z += (double)a[2] * qL;
            W.x += (double)a[3] * qA; W.y += (double)a[4] * qA; W.z += (double)a[5] * qA;
            if (BAD_GET(t)) { V.x = __longlong_as_double(0x7FF8000000000000LL); }
        }
        st4g(&vout[p0 + t], V);
        st4g(&wout[p0 + t], W);
    }
}

#undef SIG
#undef BAD_SET
#undef BAD_GET
void launch_sweep_items(bool impact, int64_t N, const double4 *vin, const double4 *win, const double *rad, double4 *vout,
                        double4 *wout, const SweepPlan &pl, const CRec *rec, const PRec *Pin, PRec *Pout,
                        const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s)
{
    if (!N) return;
    constexpr int dyn = (int)sizeof(StageBuf) + 3 * SLOT_CAP * (int)sizeof(longlong2);
    static const bool attr = [] {
        cudaFuncSetAttribute(k_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        cudaFuncSetAttribute(k_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        // shared-memory carveout (percent of the unified L1/shared capacity; unset: the driver's choice)
        if (const char *cv = getenv("DEM_SWEEP_CARVEOUT")) {
            cudaFuncSetAttribute(k_sweep<true>, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
            cudaFuncSetAttribute(k_sweep<false>, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
        }
        if (getenv("DEM_DEBUG")) {
            int per = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sweep<false>, TT, dyn);
            fprintf(stderr, "k_sweep: %d B dynamic smem, %d CTAs per SM\n", dyn, per);
        }
        return true;
    }();
    (void)attr;
    const unsigned ntiles = (unsigned)((N + TT - 1) / TT);
    if (impact)
        k_sweep<true><<<ntiles, TT, dyn, s>>>(N, vin, win, rad, vout, wout, pl.istart, pl.pin, rec, Pin, Pout, bnd,
                                              pl.wrange, sp);
    else
        k_sweep<false><<<ntiles, TT, dyn, s>>>(N, vin, win, rad, vout, wout, pl.istart, pl.pin, rec, Pin, Pout, bnd,
                                               pl.wrange, sp);
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
                            uint32_t *__restrict__ item_meta, uint16_t *__restrict__ item_own)
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
        item_own[o] = (uint16_t)(i - tb);
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
__global__ void k_plan_warps(int64_t N, const uint32_t *__restrict__ istart, uint32_t *__restrict__ wrange);
void plan_fill(int64_t N, const uint32_t *inc_start, const uint2 *inc, const double4 *pos, const SweepPlan &pl,
               cudaStream_t s, long long *launches)
{
    if (!N) return;
    k_plan_fill<<<IGRID(N)>>>(N, inc_start, inc, pl.noint, pl.istart, pl.slot_of, pl.item_c, pl.item_meta,
                              pl.item_own);
    k_plan_warps<<<(unsigned)((N + TT - 1) / TT), 32, 0, s>>>(N, pl.istart, pl.wrange);
    k_radius<<<IGRID(N)>>>(N, pos, pl.rad);
    *launches += 3;
}

// The sweep's warp ranges of each tile: warp q takes the items of whole particles from the first
// particle whose items start at or after q/NWT of the tile's items (balanced by items, so the
// tile's final barrier does not wait on a warp of coarse particles).
__global__ void __launch_bounds__(TT) k_plan_warps(int64_t N, const uint32_t *__restrict__ istart,
                                                   uint32_t *__restrict__ wrange)
{
    const int t = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * TT;
    const int np = (int)min((int64_t)TT, N - p0);
    if (t > NWT) return;
    const uint32_t I0 = istart[p0], I1 = istart[p0 + np];
    int lo = 0, hi = np;
    if (t == 0) hi = 0;
    else if (t == NWT) lo = np;
    else {
        const uint32_t tgt = I0 + (uint32_t)(((uint64_t)(I1 - I0) * (uint32_t)t + NWT - 1) / NWT);
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (istart[p0 + mid] < tgt) lo = mid + 1; else hi = mid; }
    }
    wrange[(size_t)blockIdx.x * (NWT + 1) + t] = istart[p0 + lo];
}

// ------------------------------------------------------------------ per stage: records in, impulses out
__global__ void k_item_pack(int64_t n, const uint32_t *__restrict__ item_c, const uint32_t *__restrict__ item_meta,
                            const uint16_t *__restrict__ item_own,
                            const G4 *__restrict__ geo, const double *__restrict__ cdel, const R4 *__restrict__ row,
                            const P4 *__restrict__ Pa, const P4 *__restrict__ Pb, CRec *__restrict__ rec,
                            PRec *__restrict__ P)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t c = item_c[k], meta = item_meta[k];
    const G4 g = geo[c];
    reinterpret_cast<double4 *>(rec)[k] = crec_encode(mk(g.x, g.y, g.z), cdel[c], meta, item_own[k]);
    double4 *q = reinterpret_cast<double4 *>(P + k);
    const double b = row[c].y;
    if (Pa) {
        const P4 a = Pa[c], bb = Pb[c];
        q[0] = make_double4(a.x, a.y, a.z, a.w);
        q[1] = make_double4(bb.x, bb.y, bb.z, b);
    } else {
        q[0] = make_double4(0.0, 0.0, 0.0, 0.0);
        q[1] = make_double4(0.0, 0.0, 0.0, b);
    }
}
// the stage's final impulses back to the contact arrays (one item per contact writes: body a's)
__global__ void k_item_unpack(int64_t n, const uint32_t *__restrict__ item_c, const CRec *__restrict__ rec,
                              const PRec *__restrict__ P, P4 *__restrict__ Pa, P4 *__restrict__ Pb)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    if (crec_meta(reinterpret_cast<const double4 *>(rec)[k]) & IT_B) return;
    const double4 *q = reinterpret_cast<const double4 *>(P + k);
    const double4 a = q[0], b = q[1];
    const uint32_t c = item_c[k];
    Pa[c] = mkP4(a.x, a.y, a.z, a.w);
    Pb[c] = mkP4(b.x, b.y, b.z, 0.0);
}
void item_pack(int64_t n, const SweepPlan &pl, const G4 *geo, const double *cdel, const R4 *row, const P4 *Pa,
               const P4 *Pb, CRec *rec, PRec *P, cudaStream_t s)
{ if (n) k_item_pack<<<IGRID(n)>>>(n, pl.item_c, pl.item_meta, pl.item_own, geo, cdel, row, Pa, Pb, rec, P); }
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
    flag[k] = ((m & (IT_EXT | IT_INTRA)) == IT_EXT && (m & PARTNER_PLATE) && (!own || own[cij[item_c[k]].x])) ? 1u : 0u;
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
    const double4 o = reinterpret_cast<const double4 *>(pout + k)[0];
    const int q = (item_meta[k] >> 4) & 0xF;
    const G4 g = geo[item_c[k]];
    double4 i = make_double4(0.0, 0.0, 0.0, 0.0);
    if (pin) i = reinterpret_cast<const double4 *>(pin + k)[0];
    const double dPn = o.x - i.x;
    const double d[3] = {dPn * g.x + (o.y - i.y), dPn * g.y + (o.z - i.z), dPn * g.z + (o.w - i.w)};
    for (int k2 = 0; k2 < 3; k2++) atomicAdd(&acc[3 * q + k2], (unsigned long long)llrint(d[k2] * HUB_SCALE));
}
void launch_plate_hub_items(int64_t n, const uint32_t *list, const SweepPlan &pl, const G4 *geo, const CRec *rec,
                            const PRec *pin, const PRec *pout, unsigned long long *acc, cudaStream_t s)
{ if (n) k_plate_hub_items<<<IGRID(n)>>>(n, list, pl.item_c, pl.item_meta, geo, rec, pin, pout, acc); }
#undef IGRID
