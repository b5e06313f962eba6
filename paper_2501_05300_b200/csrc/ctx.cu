// ctx.cu -- host runtime of libdem.so: the dem_ctx (device buffers, stream, rebuild policy,
// step orchestration) and the C-ABI of include/dem.h.
//
// One step:
//   [rebuild if the Verlet skin is used up]  keys -> radix sort -> permute -> per-level cell
//                                            tables -> multi-level broad phase -> transposed
//                                            lists -> history carry by sorted key
//   narrow phase (exact fp64 predicate) -> scan -> compaction + warm start -> incidence CSR
//   -> mass-splitting weights -> impact trigger -> [impact stage: N_imp Jacobi sweeps]
//   -> SPOOK rows -> gravity + warm start -> N_it Jacobi sweeps -> integrate -> plates/walls
//   -> rollback on NaN -> history scatter to the candidate slots
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dem.h"
#include "common.cuh"
#include "kernels.h"
#include "dist.h"

static thread_local std::string g_create_err;

struct dem_ctx {
    dem_material mat{};
    dem_solver sol{};
    dem_box box{};
    cudaStream_t s = nullptr;
    bool own_stream = false;
    void *(*ualloc)(size_t, void *) = nullptr;
    void (*ufree)(void *, void *) = nullptr;
    void *actx = nullptr;
    std::string err;
    std::vector<void *> allocs;

    int64_t N = 0;
    GridParams grid{};
    SolveParams sp{};
    int nlev = 1;
    double rmax_lv[DEM_MAX_LEVELS] = {0};
    bool lv_present[DEM_MAX_LEVELS] = {false};

    // particles (sorted order)
    double4 *pos = nullptr, *vel[2] = {nullptr, nullptr}, *ang[2] = {nullptr, nullptr};
    // *_prev: the state at the step start (rollback); outside that window they are scratch (the
    // rebuild's permutation target, the force evaluation, the sweep benchmark)
    double4 *xref = nullptr, *pos_prev = nullptr, *vel_prev = nullptr, *ang_prev = nullptr;
    uint32_t *gid = nullptr, *gid2 = nullptr, *gid_sorted = nullptr;
    int cur = 0;
    // sort / scan scratch
    int64_t cap_keys = 0;
    uint64_t *keys[2] = {nullptr, nullptr};
    uint32_t *vals[2] = {nullptr, nullptr};
    void *sort_tmp = nullptr;
    void *scan_tmp = nullptr;
    double *ke_part = nullptr;
    unsigned long long *lvbox = nullptr;   // per level: min xyz, max xyz (ordered bits), count
    // cells
    uint64_t ncells = 0, cap_cells = 0;
    uint32_t *cstart = nullptr, *cend = nullptr;
    // candidates
    int64_t ncand = 0, cap_cand = 0, cap_c = 0;   // candidate / contact capacities
    uint2 *cand = nullptr;
    uint32_t *co_start = nullptr, *ct_cnt = nullptr, *ct_start = nullptr, *ct_cursor = nullptr, *ct_list = nullptr;
    P4 *Pca = nullptr, *Pcb = nullptr;
    uint32_t *cflag = nullptr, *cscan = nullptr;
    // contacts
    int64_t nc = 0;
    uint2 *cij = nullptr;
    G4 *geo = nullptr;
    R4 *row = nullptr, *row_imp = nullptr;
    double *cdel = nullptr;
    P4 *Pwa = nullptr, *Pwb = nullptr;            // warm start
    P4 *Pa[2] = {nullptr, nullptr}, *Pb[2] = {nullptr, nullptr};   // [0] only (the final impulses)
    P4 *Pfa = nullptr, *Pfb = nullptr;            // final impulses of the last step
    uint32_t *ccand = nullptr;
    // incidence
    uint32_t *inc_cnt = nullptr, *inc_start = nullptr;
    // contact-once tile plan of the Jacobi sweep (sweep.cu), rebuilt every step
    SweepPlan pl{};
    uint32_t *pl_nitem = nullptr, *pl_nin = nullptr;
    unsigned int *pl_full = nullptr;
    int64_t n_items = 0, cap_items = 0;
    CRec *it_rec = nullptr;
    PRec *it_P[2] = {nullptr, nullptr};
    uint32_t *it_flag = nullptr, *it_scan = nullptr, *it_plist = nullptr;   // monolithic plates: plate items
    int64_t n_it_plist = 0;
    // CUDA graphs of the sweep loops (single context): re-captured when a pointer, the particle
    // count, the sweep count, the start parity or the solver parameters change
    struct SweepGraph { cudaGraphExec_t exec = nullptr; std::vector<unsigned char> key; };
    SweepGraph g_imp[4], g_main[4];   // small LRU caches (start parity, ping-pong pointer sets)
    int64_t g_tick = 0;
    int64_t g_used[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    uint2 *inc = nullptr;
    // history
    int64_t nh = 0, cap_h = 0;
    uint64_t *hkey = nullptr;
    P4 *hPa = nullptr, *hPb = nullptr;
    uint8_t *hauth = nullptr;       // decomposed: this rank owned a body of the history entry
    bool hist_pending = false;
    // boundary
    DevBoundary hb{};
    DevBoundary *db = nullptr;
    unsigned long long *pacc = nullptr;
    unsigned int *pcount = nullptr;
    unsigned long long *dscr_bad = nullptr;
    // monolithic plates (R18b): the step's owned plate contacts and the per-sweep impulse sums
    uint32_t *plist = nullptr;
    int64_t n_plist = 0;
    unsigned long long *hub_acc = nullptr;
    StepScalars *dsc = nullptr, *hsc = nullptr;
    uint32_t *hnc = nullptr;
    // status
    int64_t step = 0;
    bool need_rebuild = true;
    bool have_step = false;
    dem_step_report last{};
    // x-slab decomposition: owned particles [0, N_own), ghosts after
    int rank = 0, G = 1;
    Transport *tp = nullptr;
    double slab_lo = -INFINITY, slab_hi = INFINITY, band_w = 0.0;
    int64_t N_own = 0, capN = 0;
    uint8_t *own = nullptr;      // per local particle: 1 owned, 0 ghost (world_size > 1 only)
    int64_t n_send[2] = {0, 0}, n_recv[2] = {0, 0}, cap_halo[2] = {0, 0};
    uint32_t *send_pre[2] = {nullptr, nullptr}, *send_idx[2] = {nullptr, nullptr}, *recv_idx[2] = {nullptr, nullptr};
    double4 *hs[2] = {nullptr, nullptr}, *hr[2] = {nullptr, nullptr};
    // coloured Gauss-Seidel ordering (solver.ordering == 1; gs.cu)
    uint64_t *gs_key = nullptr;
    int *gs_col = nullptr;
    uint32_t *gs_ord = nullptr;
    uint2 *gs_cij = nullptr;        // contact records in colour order (coalesced per colour)
    G4 *gs_geo = nullptr;
    R4 *gs_row = nullptr;
    P4 *gs_Pa = nullptr, *gs_Pb = nullptr;
    unsigned int *gs_scr = nullptr;
    std::vector<uint32_t> gs_cstart;
    // timing
    bool timing = false;
    cudaEvent_t ev[8] = {};
    dem_timing tm{};
    long long launches = 0;
};

// ------------------------------------------------------------------ helpers
#define OWN(ctx) ((ctx)->tp ? (const uint8_t *)(ctx)->own : (const uint8_t *)nullptr)
#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);            \
            return DEM_ERR_CUDA;                                                      \
        }                                                                             \
    } while (0)
#define TRY(x)                         \
    do {                               \
        dem_status st_ = (x);          \
        if (st_ != DEM_OK) return st_; \
    } while (0)

static dem_status dalloc(dem_ctx *ctx, void **p, size_t bytes)
{
    bytes = std::max<size_t>(bytes, 256);
    bytes = (bytes + 255) & ~(size_t)255;
    void *q = nullptr;
    if (ctx->ualloc) q = ctx->ualloc(bytes, ctx->actx);
    else if (cudaMalloc(&q, bytes) != cudaSuccess) q = nullptr;
    if (!q) {
        cudaGetLastError();
        ctx->err = "device allocation of " + std::to_string(bytes) + " bytes failed";
        return DEM_ERR_OOM;
    }
    ctx->allocs.push_back(q);
    *p = q;
    return DEM_OK;
}
static void dfree(dem_ctx *ctx, void *p);
static void *ctx_alloc(size_t bytes, void *c)
{
    void *p = nullptr;
    return dalloc((dem_ctx *)c, &p, bytes) == DEM_OK ? p : nullptr;
}
static void dfree(dem_ctx *ctx, void *p)
{
    if (!p) return;
    auto it = std::find(ctx->allocs.begin(), ctx->allocs.end(), p);
    if (it != ctx->allocs.end()) ctx->allocs.erase(it);
    if (ctx->ufree) ctx->ufree(p, ctx->actx);
    else cudaFree(p);
}
template <class T>
static dem_status A(dem_ctx *ctx, T **p, size_t n)
{
    void *q = nullptr;
    TRY(dalloc(ctx, &q, n * sizeof(T)));
    *p = (T *)q;
    return DEM_OK;
}
template <class T>
static dem_status regrow(dem_ctx *ctx, T **p, size_t n)
{
    dfree(ctx, *p);
    *p = nullptr;
    return A(ctx, p, n);
}

static void tstart(dem_ctx *ctx, int k)
{
    if (ctx->timing) cudaEventRecord(ctx->ev[k], ctx->s);
}
static float telapsed(dem_ctx *ctx, int a, int b)
{
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[a], ctx->ev[b]);
    return ms;
}

// ------------------------------------------------------------------ validation and setup
static bool valid_material(const dem_material &m)
{
    return m.density > 0 && m.youngs > 0 && m.poisson >= 0 && m.poisson < 0.5 && m.mu_t >= 0 && m.mu_r >= 0 &&
           m.restitution >= 0 && m.restitution <= 1;
}

static void setup_solve_params(dem_ctx *ctx)
{
    SolveParams &sp = ctx->sp;
    const dem_solver &so = ctx->sol;
    ctx->hb.mono = so.plate_coupling == 1 ? 1 : 0;
    sp.h = so.dt;
    sp.Ups = 1.0 / (1.0 + 4.0 * so.damping_steps);
    sp.e_H = so.hertz_exp;
    sp.k_lin = so.k_lin;
    sp.Es = 1.0 / (2.0 * (1.0 - ctx->mat.poisson * ctx->mat.poisson) / ctx->mat.youngs);
    sp.rho = ctx->mat.density;
    sp.mu_t = ctx->mat.mu_t;
    sp.mu_r = ctx->mat.mu_r;
    sp.e_rest = ctx->mat.restitution;
    const double gn = std::sqrt(so.gravity[0] * so.gravity[0] + so.gravity[1] * so.gravity[1] + so.gravity[2] * so.gravity[2]);
    sp.v_imp = so.v_impact < 0 ? 20.0 * gn * so.dt : so.v_impact;
    for (int k = 0; k < 3; k++) sp.g[k] = so.gravity[k];
    sp.rolling_dims = so.rolling_dims == 2 ? 2 : 3;
    sp.hertz = so.hertz_exp == 1.0 ? 0 : 1;
    sp.Cs = sp.hertz ? 12.0 * sp.Ups / (sp.h * sp.h * sp.e_H * sp.Es) : 4.0 * sp.Ups / (sp.h * sp.h * sp.e_H * sp.k_lin);
}

// radii -> levels (factor-2 size classes), per-level r_max, skin
static dem_status setup_levels(dem_ctx *ctx, const std::vector<double> &r)
{
    double rmin = INFINITY, rmax = 0;
    for (double x : r) { rmin = std::min(rmin, x); rmax = std::max(rmax, x); }
    if (ctx->tp) {
        // every rank takes the same size classes, skin and ghost band (global radius range)
        double v[2] = {-rmin, rmax};
        if (!ctx->tp->allreduce_f64(v, 2, 1, ctx->s, ctx->err)) return DEM_ERR_NCCL;
        rmin = -v[0];
        rmax = v[1];
    }
    if (!(rmin <= rmax)) { rmin = 1e-3; rmax = 1e-3; }
    int nlev = 1;
    double t = rmin;
    while (nlev < DEM_MAX_LEVELS && rmax >= t * 2.0) { t *= 2.0; nlev++; }
    ctx->nlev = nlev;
    for (int L = 0; L < DEM_MAX_LEVELS; L++) { ctx->rmax_lv[L] = 0; ctx->lv_present[L] = false; }
    for (double x : r) {
        int L = level_of(x, rmin, nlev);
        ctx->rmax_lv[L] = std::max(ctx->rmax_lv[L], x);
        ctx->lv_present[L] = true;
    }
    if (ctx->tp) {
        // cell sizes from the global per-level maxima: ghosts and migrants of any size class fit
        if (!ctx->tp->allreduce_f64(ctx->rmax_lv, DEM_MAX_LEVELS, 1, ctx->s, ctx->err)) return DEM_ERR_NCCL;
        for (int L = 0; L < DEM_MAX_LEVELS; L++) ctx->lv_present[L] = ctx->rmax_lv[L] > 0.0;
    }
    ctx->grid.nlev = nlev;
    ctx->grid.rmin = rmin;
    ctx->grid.skin = ctx->sol.skin > 0 ? ctx->sol.skin : 0.1 * rmin;
    // ghost band: any partner of an owned particle within r_a + r_b + skin, plus one skin of margin
    // so that pairs about to meet carry their history across the faces
    ctx->band_w = 2.0 * rmax + 2.0 * ctx->grid.skin;
    if (ctx->tp) {
        // ghosts come from the two neighbouring slabs only: an interior slab must be at least one
        // band wide (decided collectively, so every rank fails the create together)
        double thin = (ctx->rank > 0 && ctx->rank < ctx->G - 1 && ctx->slab_hi - ctx->slab_lo < ctx->band_w) ? 1.0 : 0.0;
        if (!ctx->tp->allreduce_f64(&thin, 1, 1, ctx->s, ctx->err)) return DEM_ERR_NCCL;
        if (thin > 0.0) {
            ctx->err = "an interior slab is thinner than the ghost band 2 r_max + 2 skin";
            return DEM_ERR_INVALID;
        }
    }
    return DEM_OK;
}

static void setup_walls(dem_ctx *ctx)
{
    DevBoundary &b = ctx->hb;
    for (int w = 0; w < 6; w++) {
        const int ax = w / 2, side = w % 2;
        for (int k = 0; k < 3; k++) { b.wp[w][k] = 0; b.wn[w][k] = 0; }
        b.wp[w][ax] = side == 0 ? ctx->box.lo[ax] : ctx->box.hi[ax];
        b.wn[w][ax] = side == 0 ? 1.0 : -1.0;
        b.wvel[w] = 0;
        b.wpresent[w] = (ctx->box.wall_mask >> w) & 1;
        for (int k = 0; k < 3; k++) b.wforce[w][k] = 0;
        b.wcount[w] = 0;
        for (int k = 0; k < 3; k++) b.wp_ref[w][k] = b.wp[w][k];
    }
    b.wall_mu_t = ctx->box.wall_mu_t;
    b.wall_mu_r = ctx->box.wall_mu_r;
}

static dem_status upload_boundary(dem_ctx *ctx)
{
    CK(cudaMemcpyAsync(ctx->db, &ctx->hb, sizeof(DevBoundary), cudaMemcpyHostToDevice, ctx->s));
    return DEM_OK;
}

// (re)allocate the particle-sized arrays for capacity cap (contents are not preserved)
static dem_status alloc_particles(dem_ctx *ctx, int64_t cap)
{
    double4 **d4[] = {&ctx->pos, &ctx->vel[0], &ctx->vel[1], &ctx->ang[0], &ctx->ang[1], &ctx->xref, &ctx->pos_prev,
                      &ctx->vel_prev, &ctx->ang_prev};
    uint32_t **u4[] = {&ctx->gid, &ctx->gid2, &ctx->gid_sorted, &ctx->co_start, &ctx->ct_cnt, &ctx->ct_start,
                       &ctx->ct_cursor, &ctx->inc_cnt, &ctx->inc_start, &ctx->pl.istart, &ctx->pl.pin,
                       &ctx->pl_nitem, &ctx->pl_nin};
    const size_t N = (size_t)cap + 1;
    for (auto q : d4) { dfree(ctx, *q); *q = nullptr; TRY(A(ctx, q, N)); }
    // + 8 / + 2: the sweep's TMA copies of a tile's istart, pin and radii round up to 16 bytes
    for (auto q : u4) { dfree(ctx, *q); *q = nullptr; TRY(A(ctx, q, N + 8)); }
    dfree(ctx, ctx->ke_part);
    ctx->ke_part = nullptr;
    dfree(ctx, ctx->own);
    ctx->own = nullptr;
    TRY(A(ctx, &ctx->own, N));
    TRY(A(ctx, &ctx->ke_part, N / 256 + 2));
    dfree(ctx, ctx->pl.noint);
    dfree(ctx, ctx->pl.rad);
    dfree(ctx, ctx->pl.wrange);
    ctx->pl.wrange = nullptr;
    ctx->pl.noint = nullptr;
    ctx->pl.rad = nullptr;
    TRY(A(ctx, &ctx->pl.noint, N / SWEEP_TILE + 2));
    TRY(A(ctx, &ctx->pl.rad, N + 2));
    TRY(A(ctx, &ctx->pl.wrange, (N / SWEEP_TILE + 2) * (SWEEP_TILE / 32 + 1)));
    if (!ctx->lvbox) {
        TRY(A(ctx, &ctx->lvbox, (size_t)DEM_MAX_LEVELS * 8));
        TRY(A(ctx, &ctx->db, 1));
        TRY(A(ctx, &ctx->pacc, 3 * NB_SLOTS));
        TRY(A(ctx, &ctx->pcount, NB_SLOTS));
        TRY(A(ctx, &ctx->hub_acc, 3 * DEM_MAX_PLATES));
        CK(cudaMemsetAsync(ctx->hub_acc, 0, 3 * DEM_MAX_PLATES * sizeof(unsigned long long), ctx->s));
        TRY(A(ctx, &ctx->dsc, 1));
        TRY(A(ctx, &ctx->pl_full, 1));
    }
    ctx->capN = cap;
    // the key/scan scratch is not reset: it also serves the candidate and history sorts
    // (ensure_cand sized it to cap_cand, which a particle reallocation leaves unchanged)
    return DEM_OK;
}

static dem_status ensure_keys(dem_ctx *ctx, int64_t n)
{
    if (n <= ctx->cap_keys) return DEM_OK;
    int64_t cap = std::max<int64_t>(n + n / 2, 1024);
    for (int k = 0; k < 2; k++) { TRY(regrow(ctx, &ctx->keys[k], cap)); TRY(regrow(ctx, &ctx->vals[k], cap)); }
    void *p = ctx->sort_tmp;
    dfree(ctx, p);
    TRY(dalloc(ctx, &ctx->sort_tmp, sort_temp_bytes(cap)));
    dfree(ctx, ctx->scan_tmp);
    TRY(dalloc(ctx, &ctx->scan_tmp, scan_temp_bytes(cap + 1) + scan_temp_bytes(2 * cap + 2)));
    ctx->cap_keys = cap;
    return DEM_OK;
}

static dem_status ensure_cand(dem_ctx *ctx, int64_t n)
{
    if (n <= ctx->cap_cand) return DEM_OK;
    int64_t cap = std::max<int64_t>(n + n / 4, 1024);
    TRY(regrow(ctx, &ctx->cand, cap)); TRY(regrow(ctx, &ctx->ct_list, cap));
    TRY(regrow(ctx, &ctx->Pca, cap)); TRY(regrow(ctx, &ctx->Pcb, cap));
    TRY(regrow(ctx, &ctx->cflag, cap + 1)); TRY(regrow(ctx, &ctx->cscan, cap + 1));
    if (!ctx->gs_scr) TRY(A(ctx, &ctx->gs_scr, 260));
    ctx->cap_cand = cap;
    ctx->nc = 0;
    ctx->have_step = false;
    return ensure_keys(ctx, std::max<int64_t>(cap, ctx->N));
}

// the contact-indexed arrays, sized by the contact count of the step (about half the candidates
// with the Verlet skin) rather than by the candidates; contents are dead at the point of call
// (before the compaction), so a regrow keeps nothing
static dem_status ensure_contacts(dem_ctx *ctx, int64_t n)
{
    if (n <= ctx->cap_c) return DEM_OK;
    int64_t cap = std::max<int64_t>(n + n / 4, 1024);
    TRY(regrow(ctx, &ctx->cij, cap)); TRY(regrow(ctx, &ctx->geo, cap)); TRY(regrow(ctx, &ctx->row, cap)); TRY(regrow(ctx, &ctx->cdel, cap));
    TRY(regrow(ctx, &ctx->row_imp, cap)); TRY(regrow(ctx, &ctx->Pwa, cap)); TRY(regrow(ctx, &ctx->Pwb, cap));
    TRY(regrow(ctx, &ctx->Pa[0], cap)); TRY(regrow(ctx, &ctx->Pb[0], cap));   // final impulses, contact order
    ctx->Pfa = ctx->Pa[0];
    ctx->Pfb = ctx->Pb[0];
    TRY(regrow(ctx, &ctx->ccand, cap));
    TRY(regrow(ctx, &ctx->pl.slot_of, cap));
    TRY(regrow(ctx, &ctx->plist, cap + 1));
    if (ctx->sol.ordering == 1 || ctx->gs_cij) {   // Gauss-Seidel buffers only when that ordering is used
        TRY(regrow(ctx, &ctx->gs_key, cap)); TRY(regrow(ctx, &ctx->gs_col, cap)); TRY(regrow(ctx, &ctx->gs_ord, cap));
        TRY(regrow(ctx, &ctx->gs_cij, cap)); TRY(regrow(ctx, &ctx->gs_geo, cap)); TRY(regrow(ctx, &ctx->gs_row, cap));
        TRY(regrow(ctx, &ctx->gs_Pa, cap)); TRY(regrow(ctx, &ctx->gs_Pb, cap));
    }
    TRY(regrow(ctx, &ctx->inc, 2 * cap));
    ctx->cap_c = cap;
    return DEM_OK;
}

// ------------------------------------------------------------------ level bounding boxes
__device__ __forceinline__ unsigned long long ord_bits(double x)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
static double ord_unbits(unsigned long long u)
{
    unsigned long long b = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFULL) : ~u;
    double x;
    std::memcpy(&x, &b, 8);
    return x;
}
// per-level bounding boxes and counts: shared-memory partials per block, then one global
// atomic per block and value (min/max/count are order-independent: deterministic)
__global__ void k_level_bbox(int64_t N, const double4 *__restrict__ pos, double rmin, int nlev,
                             unsigned long long *__restrict__ box)
{
    __shared__ unsigned long long sb[DEM_MAX_LEVELS * 8];
    for (int q = threadIdx.x; q < DEM_MAX_LEVELS * 8; q += blockDim.x) {
        const int f = q & 7;
        sb[q] = f < 3 ? ~0ULL : 0ULL;
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // warp-level min/max first when the warp's particles share a level (the sorted order makes
    // that the rule), so only lane 0 touches the shared box: per-thread shared atomics on the
    // same 7 words serialised the kernel (1.2 ms for 14.6 M particles)
    const bool act = i < N;
    double4 p = act ? pos[i] : make_double4(0.0, 0.0, 0.0, 0.0);
    const int L = act ? level_of(p.w, rmin, nlev) : -1;
    const int L0 = __shfl_sync(0xffffffffu, L, 0);
    if (__all_sync(0xffffffffu, L == L0) && L0 >= 0) {
        unsigned long long v[6];
        const double c[3] = {p.x, p.y, p.z};
        for (int k = 0; k < 3; k++) { v[k] = ord_bits(c[k]); v[3 + k] = v[k]; }
        for (int o = 16; o; o >>= 1)
            for (int k = 0; k < 3; k++) {
                v[k] = min(v[k], __shfl_xor_sync(0xffffffffu, v[k], o));
                v[3 + k] = max(v[3 + k], __shfl_xor_sync(0xffffffffu, v[3 + k], o));
            }
        if ((threadIdx.x & 31) == 0) {
            unsigned long long *b = sb + 8 * L0;
            for (int k = 0; k < 3; k++) { atomicMin(&b[k], v[k]); atomicMax(&b[3 + k], v[3 + k]); }
            atomicAdd(&b[6], 32ULL);
        }
    } else if (act) {
        unsigned long long *b = sb + 8 * L;
        const double c[3] = {p.x, p.y, p.z};
        for (int k = 0; k < 3; k++) {
            atomicMin(&b[k], ord_bits(c[k]));
            atomicMax(&b[3 + k], ord_bits(c[k]));
        }
        atomicAdd(&b[6], 1ULL);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nlev * 8; q += blockDim.x) {
        const int f = q & 7;
        if (sb[8 * (q >> 3) + 6] == 0 || f == 7) continue;
        if (f < 3) atomicMin(&box[q], sb[q]);
        else if (f < 6) atomicMax(&box[q], sb[q]);
        else atomicAdd(&box[q], sb[q]);
    }
}

static dem_status compute_grid(dem_ctx *ctx)
{
    std::vector<unsigned long long> hb(8 * DEM_MAX_LEVELS);
    for (int L = 0; L < DEM_MAX_LEVELS; L++) {
        for (int k = 0; k < 3; k++) { hb[8 * L + k] = ~0ULL; hb[8 * L + 3 + k] = 0ULL; }
        hb[8 * L + 6] = 0;
        hb[8 * L + 7] = 0;
    }
    CK(cudaMemcpyAsync(ctx->lvbox, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice, ctx->s));
    if (ctx->N) {
        k_level_bbox<<<(unsigned)((ctx->N + 255) / 256), 256, 0, ctx->s>>>(ctx->N, ctx->pos, ctx->grid.rmin, ctx->nlev, ctx->lvbox);
        ctx->launches++;
    }
    CK(cudaMemcpyAsync(hb.data(), ctx->lvbox, hb.size() * 8, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    GridParams &g = ctx->grid;
    uint64_t off = 0;
    int bits = 1;
    for (int L = 0; L < ctx->nlev; L++) {
        GridLevel &lv = g.lv[L];
        lv.present = hb[8 * L + 6] > 0;
        lv.rmax = ctx->rmax_lv[L];
        lv.cell = 2.0 * lv.rmax + g.skin;
        if (!lv.present) { lv.nx = lv.ny = lv.nz = 1; lv.offset = off; lv.ox = lv.oy = lv.oz = 0; continue; }
        double lo[3], hi[3];
        for (int k = 0; k < 3; k++) { lo[k] = ord_unbits(hb[8 * L + k]); hi[k] = ord_unbits(hb[8 * L + 3 + k]); }
        // coarser-level queries come from finer particles anywhere: extend by the global box
        for (int k = 0; k < 3; k++) {
            if (!std::isfinite(lo[k]) || !std::isfinite(hi[k])) { ctx->err = "non-finite particle position"; return DEM_ERR_DIVERGED; }
        }
        int n[3];
        double o[3];
        for (int k = 0; k < 3; k++) {
            o[k] = lo[k] - lv.cell;
            double ext = (hi[k] - lo[k]) + 2.0 * lv.cell;
            long long nn = (long long)std::ceil(ext / lv.cell) + 1;
            nn = std::max<long long>(1, std::min<long long>(nn, 1 << 20));
            n[k] = (int)nn;
        }
        lv.ox = o[0]; lv.oy = o[1]; lv.oz = o[2];
        lv.nx = n[0]; lv.ny = n[1]; lv.nz = n[2];
        lv.offset = off;
        off += (uint64_t)n[0] * n[1] * n[2];
        for (int k = 0; k < 3; k++) while ((1 << bits) < n[k]) bits++;
    }
    for (int L = ctx->nlev; L < DEM_MAX_LEVELS; L++) g.lv[L].present = 0;
    g.bits = bits;
    if (getenv("DEM_DEBUG")) {
        for (int L = 0; L < ctx->nlev; L++)
            fprintf(stderr, "[dem r%d N=%lld own=%lld] level %d cell %.6g n %d %d %d o %.6g %.6g %.6g bits %d rmax %.6g\n",
                    ctx->rank, (long long)ctx->N, (long long)ctx->N_own, L, g.lv[L].cell, g.lv[L].nx, g.lv[L].ny,
                    g.lv[L].nz, g.lv[L].ox, g.lv[L].oy, g.lv[L].oz, bits, g.lv[L].rmax);
    }
    ctx->ncells = off;
    if (off > ctx->cap_cells) {
        uint64_t cap = off + off / 4 + 64;
        TRY(regrow(ctx, &ctx->cstart, cap));
        TRY(regrow(ctx, &ctx->cend, cap));
        ctx->cap_cells = cap;
    }
    return DEM_OK;
}

// ------------------------------------------------------------------ rebuild
static dem_status export_history(dem_ctx *ctx)
{
    const int64_t nc = ctx->ncand;
    cudaStream_t s = ctx->s;
    ctx->nh = 0;
    if (!nc) return DEM_OK;
    launch_hist_flag(nc, ctx->Pca, ctx->Pcb, ctx->cflag, s);
    scan_u32(ctx->cflag, ctx->cscan, nc, ctx->scan_tmp, s, &ctx->launches);
    uint32_t nh = 0;
    CK(cudaMemcpyAsync(&nh, ctx->cscan + nc, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx->launches += 1;
    if (nh > ctx->cap_h) {
        int64_t cap = nh + nh / 4 + 1024;
        TRY(regrow(ctx, &ctx->hkey, cap)); TRY(regrow(ctx, &ctx->hPa, cap)); TRY(regrow(ctx, &ctx->hPb, cap));
        TRY(regrow(ctx, &ctx->hauth, cap));
        ctx->cap_h = cap;
    }
    if (nh) {
        launch_hist_keys(nc, ctx->cflag, ctx->cscan, ctx->cand, ctx->gid, ctx->keys[0], ctx->vals[0], s);
        radix_sort_u64(ctx->keys, ctx->vals, nh, 64, ctx->sort_tmp, s, &ctx->launches);
        CK(cudaMemcpyAsync(ctx->hkey, ctx->keys[0], nh * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
        launch_hist_gather(nh, ctx->vals[0], ctx->cand, ctx->gid, ctx->Pca, ctx->Pcb, ctx->hPa, ctx->hPb, s);
        if (ctx->tp) launch_hist_auth(nh, ctx->vals[0], ctx->cand, ctx->own, ctx->hauth, s);
        ctx->launches += ctx->tp ? 3 : 2;
    }
    ctx->nh = nh;
    if (getenv("DEM_DEBUG")) fprintf(stderr, "[dem r%d] export history: ncand %lld nh %u\n", ctx->rank, (long long)nc, nh);
    return DEM_OK;
}

// ------------------------------------------------------------------ x-slab decomposition
static dem_status grow_halo(dem_ctx *ctx, int k, int64_t n)
{
    if (n <= ctx->cap_halo[k]) return DEM_OK;
    const int64_t cap = n + n / 4 + 256;
    TRY(regrow(ctx, &ctx->send_pre[k], cap)); TRY(regrow(ctx, &ctx->send_idx[k], cap)); TRY(regrow(ctx, &ctx->recv_idx[k], cap));
    TRY(regrow(ctx, &ctx->hs[k], 4 * cap)); TRY(regrow(ctx, &ctx->hr[k], 4 * cap));
    ctx->cap_halo[k] = cap;
    return DEM_OK;
}

static dem_status xchg(dem_ctx *ctx, const void *const snd[2], const size_t sb[2], void *const rcv[2], const size_t rb[2])
{
    if (!ctx->tp->exchange(snd, sb, rcv, rb, ctx->s, ctx->err)) return DEM_ERR_NCCL;
    return DEM_OK;
}

// ghost velocities (v, c/m; w, c/I) from their owners, after every update of the velocities
static dem_status halo(dem_ctx *ctx, double4 *vel, double4 *ang)
{
    if (!ctx->tp) return DEM_OK;
    for (int k = 0; k < 2; k++) launch_pack_halo(ctx->n_send[k], ctx->send_idx[k], vel, ang, ctx->hs[k], ctx->s);
    const void *snd[2] = {ctx->hs[0], ctx->hs[1]};
    void *rcv[2] = {ctx->hr[0], ctx->hr[1]};
    const size_t sb[2] = {(size_t)ctx->n_send[0] * 64, (size_t)ctx->n_send[1] * 64};
    const size_t rb[2] = {(size_t)ctx->n_recv[0] * 64, (size_t)ctx->n_recv[1] * 64};
    TRY(xchg(ctx, snd, sb, rcv, rb));
    for (int k = 0; k < 2; k++) launch_unpack_halo(ctx->n_recv[k], ctx->recv_idx[k], ctx->hr[k], vel, ang, ctx->s);
    ctx->launches += 4;
    return DEM_OK;
}

// At a rebuild: ownership by slab, then the ghost bands of both neighbours.  A particle that
// crossed into a neighbour's slab was a ghost there with a bit-identical state (ghosts move with
// their owners' velocities), so it is simply owned there from now on: no particle is shipped
// except as a band copy.  Owned particles come first, ghosts after (left band, right band).
// History hand-over at a rebuild (dist.cu k_hist_*): after the new local sets are formed, send
// each neighbour the authoritative history entries (this rank owned a body before the rebuild)
// whose bodies the neighbour now holds -- its band from us and our band from it -- and merge the
// received entries over ours (they win for equal keys).
static dem_status exchange_history(dem_ctx *ctx, int64_t n_own, const uint32_t *tg, const uint32_t nsend[2],
                                   const unsigned long long rc[2], const int has[2])
{
    cudaStream_t s = ctx->s;
    const int64_t nh = ctx->nh;
    void *sbuf[2] = {nullptr, nullptr}, *rbuf[2] = {nullptr, nullptr};
    unsigned long long ns[2] = {0, 0}, nr[2] = {0, 0};
    uint64_t *B = nullptr;
    uint32_t *flag = nullptr, *scan = nullptr, *idx = nullptr;
    const int64_t nBmax = std::max<int64_t>((int64_t)nsend[0] + (int64_t)rc[0], (int64_t)nsend[1] + (int64_t)rc[1]);
    TRY(ensure_keys(ctx, std::max<int64_t>(nBmax, 1)));
    TRY(A(ctx, &B, nBmax + 1));
    TRY(A(ctx, &flag, nh + 2)); TRY(A(ctx, &scan, nh + 2)); TRY(A(ctx, &idx, nh + 2));
    const int64_t goff[2] = {n_own, n_own + (int64_t)rc[0]};
    for (int k = 0; k < 2; k++) {
        if (has[k] && nh) {
            const int64_t nB = (int64_t)nsend[k] + (int64_t)rc[k];
            launch_gid_list(nsend[k], ctx->send_pre[k], tg, ctx->keys[0], s);
            launch_gid_list((int64_t)rc[k], nullptr, ctx->gid + goff[k], ctx->keys[0] + nsend[k], s);
            if (nB) radix_sort_u64(ctx->keys, ctx->vals, nB, 32, ctx->sort_tmp, s, &ctx->launches);
            CK(cudaMemcpyAsync(B, ctx->keys[0], nB * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
            launch_hist_select(nh, ctx->hkey, ctx->hauth, B, nB, flag, s);
            scan_u32(flag, scan, nh, ctx->scan_tmp, s, &ctx->launches);
            uint32_t cnt = 0;
            CK(cudaMemcpyAsync(&cnt, scan + nh, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            ns[k] = cnt;
            TRY(dalloc(ctx, &sbuf[k], std::max<size_t>(cnt, 1) * HIST_REC_BYTES));
            launch_compact_idx(nh, flag, scan, idx, s);
            launch_hist_pack(cnt, idx, ctx->hkey, ctx->hPa, ctx->hPb, sbuf[k], s);
            ctx->launches += 4;
        } else {
            TRY(dalloc(ctx, &sbuf[k], HIST_REC_BYTES));
        }
    }
    {   // counts, then the records
        unsigned long long *cnt = nullptr;
        TRY(A(ctx, &cnt, 4));
        CK(cudaMemcpyAsync(cnt, ns, 16, cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(cnt + 2, 0, 16, s));
        const void *snd[2] = {cnt, cnt + 1};
        void *rcv[2] = {cnt + 2, cnt + 3};
        const size_t sb[2] = {has[0] ? 8u : 0u, has[1] ? 8u : 0u};
        TRY(xchg(ctx, snd, sb, rcv, sb));
        CK(cudaMemcpyAsync(nr, cnt + 2, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        dfree(ctx, cnt);
    }
    for (int k = 0; k < 2; k++) TRY(dalloc(ctx, &rbuf[k], std::max<size_t>(nr[k], 1) * HIST_REC_BYTES));
    {
        const void *snd[2] = {sbuf[0], sbuf[1]};
        const size_t sb[2] = {(size_t)ns[0] * HIST_REC_BYTES, (size_t)ns[1] * HIST_REC_BYTES};
        const size_t rb[2] = {(size_t)nr[0] * HIST_REC_BYTES, (size_t)nr[1] * HIST_REC_BYTES};
        TRY(xchg(ctx, snd, sb, rbuf, rb));
    }
    const int64_t total = nh + (int64_t)nr[0] + (int64_t)nr[1];
    if (total > nh) {
        // own entries then the received ones, stable-sorted by key; the last of each key is kept
        TRY(ensure_keys(ctx, total));
        P4 *ca = nullptr, *cb = nullptr;
        uint32_t *f2 = nullptr, *s2 = nullptr;
        TRY(A(ctx, &ca, total)); TRY(A(ctx, &cb, total)); TRY(A(ctx, &f2, total + 1)); TRY(A(ctx, &s2, total + 1));
        launch_iota_keys(nh, ctx->hkey, ctx->keys[0], ctx->vals[0], s);
        if (nh) {
            CK(cudaMemcpyAsync(ca, ctx->hPa, nh * sizeof(P4), cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(cb, ctx->hPb, nh * sizeof(P4), cudaMemcpyDeviceToDevice, s));
        }
        int64_t o = nh;
        for (int k = 0; k < 2; k++) {
            launch_hist_unpack((int64_t)nr[k], rbuf[k], ctx->keys[0] + o, ctx->vals[0] + o, (uint32_t)o, ca + o, cb + o, s);
            o += (int64_t)nr[k];
        }
        radix_sort_u64(ctx->keys, ctx->vals, total, 64, ctx->sort_tmp, s, &ctx->launches);
        launch_hist_last(total, ctx->keys[0], f2, s);
        scan_u32(f2, s2, total, ctx->scan_tmp, s, &ctx->launches);
        uint32_t nn = 0;
        CK(cudaMemcpyAsync(&nn, s2 + total, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if ((int64_t)nn > ctx->cap_h) {
            const int64_t cap = nn + nn / 4 + 1024;
            TRY(regrow(ctx, &ctx->hkey, cap)); TRY(regrow(ctx, &ctx->hPa, cap)); TRY(regrow(ctx, &ctx->hPb, cap));
            TRY(regrow(ctx, &ctx->hauth, cap));
            ctx->cap_h = cap;
        }
        launch_hist_emit(total, f2, s2, ctx->keys[0], ctx->vals[0], ca, cb, ctx->hkey, ctx->hPa, ctx->hPb, s);
        CK(cudaStreamSynchronize(s));
        ctx->nh = nn;
        for (void *q : {(void *)ca, (void *)cb, (void *)f2, (void *)s2}) dfree(ctx, q);
        ctx->launches += 4;
    }
    for (int k = 0; k < 2; k++) { dfree(ctx, sbuf[k]); dfree(ctx, rbuf[k]); }
    for (void *q : {(void *)B, (void *)flag, (void *)scan, (void *)idx}) dfree(ctx, q);
    if (getenv("DEM_DEBUG"))
        fprintf(stderr, "[dem r%d] history hand-over: sent %llu/%llu received %llu/%llu -> %lld entries\n", ctx->rank,
                ns[0], ns[1], nr[0], nr[1], (long long)ctx->nh);
    return DEM_OK;
}

static dem_status redistribute(dem_ctx *ctx)
{
    cudaStream_t s = ctx->s;
    const int64_t N = ctx->N;
    uint32_t *flag = nullptr, *scan = nullptr, *idx = nullptr, *tg = nullptr;
    double4 *tp = nullptr, *tv = nullptr, *tw = nullptr;
    TRY(A(ctx, &flag, N + 2)); TRY(A(ctx, &scan, N + 2)); TRY(A(ctx, &idx, N + 2)); TRY(A(ctx, &tg, N + 2));
    TRY(A(ctx, &tp, N + 1)); TRY(A(ctx, &tv, N + 1)); TRY(A(ctx, &tw, N + 1));
    // 1. owned = x in [slab_lo, slab_hi), compacted in the current order
    // the outer ranks own everything beyond the box faces too: no particle can be orphaned
    const double own_lo = ctx->rank == 0 ? -INFINITY : ctx->slab_lo;
    const double own_hi = ctx->rank == ctx->G - 1 ? INFINITY : ctx->slab_hi;
    launch_slab_flags(N, ctx->pos, own_lo, own_hi, flag, s);
    scan_u32(flag, scan, N, ctx->scan_tmp, s, &ctx->launches);
    uint32_t n_own = 0;
    CK(cudaMemcpyAsync(&n_own, scan + N, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    launch_compact_idx(N, flag, scan, idx, s);
    launch_gather_state(n_own, idx, ctx->pos, ctx->vel[ctx->cur], ctx->ang[ctx->cur], ctx->gid, tp, tv, tw, tg, s);
    // 2. bands of the owned set facing each neighbour
    const int has[2] = {ctx->rank > 0, ctx->rank < ctx->G - 1};
    uint32_t *fb[2] = {flag, idx};                    // reuse the scratch (n_own <= N)
    launch_band_flags(n_own, tp, ctx->slab_lo + ctx->band_w, ctx->slab_hi - ctx->band_w, has[0], has[1], fb[0], fb[1], s);
    uint32_t nsend[2] = {0, 0};
    uint32_t *bscan2 = nullptr;
    TRY(A(ctx, &bscan2, N + 2));
    uint32_t *bscan[2] = {scan, bscan2};
    for (int k = 0; k < 2; k++) {
        scan_u32(fb[k], bscan[k], n_own, ctx->scan_tmp, s, &ctx->launches);
        CK(cudaMemcpyAsync(&nsend[k], bscan[k] + n_own, 4, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    // 3. band sizes to the neighbours
    unsigned long long *cnt = nullptr;
    TRY(A(ctx, &cnt, 4));
    const unsigned long long hc[2] = {nsend[0], nsend[1]};
    CK(cudaMemcpyAsync(cnt, hc, 16, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(cnt + 2, 0, 16, s));
    {
        const void *snd[2] = {cnt, cnt + 1};
        void *rcv[2] = {cnt + 2, cnt + 3};
        const size_t sb[2] = {has[0] ? 8u : 0u, has[1] ? 8u : 0u};
        TRY(xchg(ctx, snd, sb, rcv, sb));
    }
    unsigned long long rc[2] = {0, 0};
    CK(cudaMemcpyAsync(rc, cnt + 2, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(ctx, cnt);
    // 4. band lists (halo buffers sized for both directions first: growing reallocates them)
    for (int k = 0; k < 2; k++) {
        TRY(grow_halo(ctx, k, std::max<int64_t>(nsend[k], (int64_t)rc[k])));
        launch_compact_idx(n_own, fb[k], bscan[k], ctx->send_pre[k], s);
        launch_pack_band(nsend[k], ctx->send_pre[k], tp, tv, tw, tg, ctx->hs[k], s);
    }
    CK(cudaStreamSynchronize(s));
    dfree(ctx, bscan2);
    {
        const void *snd[2] = {ctx->hs[0], ctx->hs[1]};
        void *rcv[2] = {ctx->hr[0], ctx->hr[1]};
        const size_t sb[2] = {(size_t)nsend[0] * 128, (size_t)nsend[1] * 128};
        const size_t rb[2] = {(size_t)rc[0] * 128, (size_t)rc[1] * 128};
        TRY(xchg(ctx, snd, sb, rcv, rb));
    }
    // 5. new local set: owned, left ghosts, right ghosts
    const int64_t Nn = (int64_t)n_own + (int64_t)rc[0] + (int64_t)rc[1];
    if (Nn > ctx->capN) {
        CK(cudaStreamSynchronize(s));
        TRY(alloc_particles(ctx, Nn + Nn / 4 + 1024));
    }
    ctx->cur = 0;
    CK(cudaMemcpyAsync(ctx->pos, tp, n_own * sizeof(double4), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ctx->vel[0], tv, n_own * sizeof(double4), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ctx->ang[0], tw, n_own * sizeof(double4), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ctx->gid, tg, n_own * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    int64_t off = n_own;
    for (int k = 0; k < 2; k++) {
        launch_unpack_band(rc[k], ctx->hr[k], ctx->pos + off, ctx->vel[0] + off, ctx->ang[0] + off, ctx->gid + off, s);
        off += rc[k];
    }
    CK(cudaStreamSynchronize(s));
    TRY(exchange_history(ctx, n_own, tg, nsend, rc, has));
    for (void *q : {(void *)flag, (void *)scan, (void *)idx, (void *)tg, (void *)tp, (void *)tv, (void *)tw}) dfree(ctx, q);
    ctx->N = Nn;
    ctx->N_own = n_own;
    for (int k = 0; k < 2; k++) { ctx->n_send[k] = nsend[k]; ctx->n_recv[k] = (int64_t)rc[k]; }
    ctx->launches += 8;
    return DEM_OK;
}

// after the rebuild's sort (perm: new -> old): owned flags, halo index lists in sorted positions,
// owned gids in order (owned and ghost particles stay interleaved in the Morton order)
static dem_status finish_decomposition(dem_ctx *ctx, const uint32_t *perm)
{
    cudaStream_t s = ctx->s;
    const int64_t N = ctx->N;
    uint32_t *inv = nullptr;
    TRY(A(ctx, &inv, N + 1));
    launch_own_flags(N, perm, (uint32_t)ctx->N_own, ctx->own, s);
    launch_inv_perm(N, perm, inv, s);
    int64_t off = ctx->N_own;
    for (int k = 0; k < 2; k++) {
        launch_map_idx(ctx->n_send[k], ctx->send_pre[k], 0u, inv, ctx->send_idx[k], s);
        launch_map_idx(ctx->n_recv[k], nullptr, (uint32_t)off, inv, ctx->recv_idx[k], s);
        off += ctx->n_recv[k];
    }
    // gid-sorted owned ids (getters report owned particles in gid order)
    if (ctx->N_own) {
        launch_gid_keys(N, ctx->gid, ctx->own, ctx->keys[0], ctx->vals[0], s);
        radix_sort_u64(ctx->keys, ctx->vals, N, 33, ctx->sort_tmp, s, &ctx->launches);
        launch_keys_to_u32(ctx->N_own, ctx->keys[0], ctx->gid_sorted, s);
    }
    CK(cudaStreamSynchronize(s));
    dfree(ctx, inv);
    ctx->launches += 6;
    return DEM_OK;
}

static dem_status sync_check(dem_ctx *ctx, const char *where)
{
    if (!getenv("DEM_SYNC_CHECK")) return DEM_OK;
    const cudaError_t e = cudaStreamSynchronize(ctx->s);
    const cudaError_t e2 = cudaGetLastError();
    if (e != cudaSuccess || e2 != cudaSuccess) {
        ctx->err = std::string("sync check at ") + where + ": " + cudaGetErrorString(e != cudaSuccess ? e : e2);
        return DEM_ERR_CUDA;
    }
    return DEM_OK;
}

// Decomposed: a failure on one rank must stop every rank before the next collective (else the
// others block in it).  The statuses are max-reduced over the ranks at each decision point;
// ranks that did not fail themselves report the failure of another.
static dem_status agree(dem_ctx *ctx, dem_status st)
{
    if (!ctx->tp) return st;
    double f = (double)(int)st;
    std::string e;
    if (!ctx->tp->allreduce_f64(&f, 1, 1, ctx->s, e)) { ctx->err = e; return DEM_ERR_NCCL; }
    const dem_status g = (dem_status)(int)f;
    if (g != DEM_OK && st == DEM_OK) ctx->err = "another rank failed (status " + std::to_string((int)g) + ")";
    return g;
}

static dem_status rebuild(dem_ctx *ctx)
{
    cudaStream_t s = ctx->s;
    TRY(sync_check(ctx, "rebuild entry"));
    if (!ctx->hist_pending) TRY(export_history(ctx));
    ctx->hist_pending = false;
    if (ctx->tp) {
        TRY(agree(ctx, ensure_keys(ctx, std::max<int64_t>(ctx->N, 1))));
        TRY(redistribute(ctx));
    } else {
        ctx->N_own = ctx->N;
    }
    const int64_t N = ctx->N;
    TRY(ensure_keys(ctx, std::max<int64_t>(N, 1)));
    TRY(compute_grid(ctx));
    // (a) level + Morton keys, stable radix sort, permutation of the SoA state
    if (N) {
        launch_keys(N, ctx->pos, ctx->grid, ctx->keys[0], ctx->vals[0], s);
        const int nbits = 3 * ctx->grid.bits + 3;
        radix_sort_u64(ctx->keys, ctx->vals, N, nbits, ctx->sort_tmp, s, &ctx->launches);
        // into the *_prev buffers (free until the step copies its start state there)
        launch_permute(N, ctx->vals[0], ctx->pos, ctx->vel[ctx->cur], ctx->ang[ctx->cur], ctx->gid, ctx->pos_prev,
                       ctx->vel_prev, ctx->ang_prev, ctx->gid2, s);
        std::swap(ctx->pos, ctx->pos_prev);
        std::swap(ctx->vel[ctx->cur], ctx->vel_prev);
        std::swap(ctx->ang[ctx->cur], ctx->ang_prev);
        std::swap(ctx->gid, ctx->gid2);
        ctx->launches += 2;
        // (b) per-level dense cell tables
        CK(cudaMemsetAsync(ctx->cstart, 0, ctx->ncells * sizeof(uint32_t), s));
        CK(cudaMemsetAsync(ctx->cend, 0, ctx->ncells * sizeof(uint32_t), s));
        launch_cells(N, ctx->keys[0], ctx->grid, ctx->cstart, ctx->cend, s);
        if (ctx->tp) TRY(finish_decomposition(ctx, ctx->vals[0]));   // reuses keys/vals after the cells
        // multi-level broad phase: count, scan, fill
        launch_broad(false, N, ctx->pos, ctx->grid, ctx->cstart, ctx->cend, ctx->db, ctx->co_start, nullptr, s);
        ctx->launches += 2;
    }
    scan_u32(ctx->co_start, ctx->co_start, N, ctx->scan_tmp, s, &ctx->launches);
    uint32_t ncand = 0;
    CK(cudaMemcpyAsync(&ncand, ctx->co_start + N, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (ncand >= CCAND_FLIP) { ctx->err = "more than 2^31 contact candidates on one rank"; return DEM_ERR_OOM; }
    TRY(ensure_cand(ctx, std::max<int64_t>(ncand, 1)));
    ctx->ncand = ncand;
    if (N) {
        launch_broad(true, N, ctx->pos, ctx->grid, ctx->cstart, ctx->cend, ctx->db, ctx->co_start, ctx->cand, s);
        ctx->launches++;
    }
    launch_trans(N, ncand, ctx->cand, ctx->ct_cnt, ctx->ct_start, ctx->ct_cursor, ctx->ct_list, ctx->scan_tmp, s,
                 &ctx->launches);
    // (c) history carried across the rebuild by sorted-key lookup
    launch_hist_carry(ncand, ctx->cand, ctx->gid, ctx->hkey, ctx->hPa, ctx->hPb, ctx->nh, ctx->Pca, ctx->Pcb, s);
    ctx->launches++;
    if (N) CK(cudaMemcpyAsync(ctx->xref, ctx->pos, N * sizeof(double4), cudaMemcpyDeviceToDevice, s));
    // boundary references (device copy is authoritative; hb mirrors it after every step)
    for (int w = 0; w < 6; w++) for (int k = 0; k < 3; k++) ctx->hb.wp_ref[w][k] = ctx->hb.wp[w][k];
    for (int q = 0; q < DEM_MAX_PLATES; q++) for (int k = 0; k < 3; k++) ctx->hb.ppos_ref[q][k] = ctx->hb.ppos[q][k];
    TRY(upload_boundary(ctx));
    ctx->need_rebuild = false;
    CK(cudaGetLastError());
    return DEM_OK;
}

// ------------------------------------------------------------------ one step
// the Jacobi sweep's tile plan of this step (sweep.cu): items per tile, slots, radii
static dem_status build_plan(dem_ctx *ctx, int64_t N)
{
    cudaStream_t s = ctx->s;
    if (N > (int64_t)IT_IDX) { ctx->err = "more than 2^29 local particles on one rank"; return DEM_ERR_INVALID; }
    plan_counts(N, ctx->inc_start, ctx->inc, ctx->pl, ctx->pl_nitem, ctx->pl_nin, ctx->pl_full, ctx->scan_tmp, s,
                &ctx->launches);
    uint32_t ni = 0;
    CK(cudaMemcpyAsync(&ni, ctx->pl.istart + N, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if ((int64_t)ni > ctx->cap_items) {
        const int64_t cap = std::max<int64_t>((int64_t)ni + ni / 4, 1024);
        TRY(regrow(ctx, &ctx->pl.item_c, cap)); TRY(regrow(ctx, &ctx->pl.item_meta, cap));
        TRY(regrow(ctx, &ctx->pl.item_own, cap));
        TRY(regrow(ctx, &ctx->it_rec, cap)); TRY(regrow(ctx, &ctx->it_P[0], cap));
        TRY(regrow(ctx, &ctx->it_P[1], cap));
        TRY(regrow(ctx, &ctx->it_flag, cap + 1)); TRY(regrow(ctx, &ctx->it_scan, cap + 1));
        TRY(regrow(ctx, &ctx->it_plist, cap + 1));
        ctx->cap_items = cap;
        TRY(ensure_keys(ctx, cap + 1));   // scan scratch of the plate-item list
    }
    ctx->n_items = ni;
    plan_fill(N, ctx->inc_start, ctx->inc, ctx->pos, ctx->pl, s, &ctx->launches);
    if (getenv("DEM_DEBUG")) {
        unsigned full = 0;
        CK(cudaMemcpyAsync(&full, ctx->pl_full, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fprintf(stderr, "[dem] sweep plan: %u items for %lld contacts (%.3f per contact)%s\n", ni, (long long)ctx->nc,
                ctx->nc ? (double)ni / ctx->nc : 0.0, full ? ", some tiles over the slot capacity" : "");
    }
    return DEM_OK;
}

// monolithic plates (R18b): the impulse the force-driven plate axes received between pin and pout
// (pin == nullptr: all of pout; first: plus the external impulse h F), summed over the ranks.
// items: pin/pout are item impulse records (sweeps), else contact-indexed P4 (warm start).
static bool mono_active(const dem_ctx *ctx) { return ctx->hb.mono && ctx->hb.n_plates > 0 && ctx->sol.ordering == 0; }
static dem_status plate_hub(dem_ctx *ctx, bool items, const void *pin, const void *pout, int first)
{
    cudaStream_t s = ctx->s;
    if (items)
        launch_plate_hub_items(ctx->n_it_plist, ctx->it_plist, ctx->pl, ctx->geo, ctx->it_rec, (const PRec *)pin,
                               (const PRec *)pout, ctx->hub_acc, s);
    else
        launch_plate_hub(ctx->n_plist, ctx->plist, ctx->cij, ctx->geo, pin, pout, ctx->hub_acc, s);
    if (ctx->tp) {
        long long v[3 * DEM_MAX_PLATES];
        CK(cudaMemcpyAsync(v, ctx->hub_acc, sizeof(v), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (!ctx->tp->allreduce_i64(v, 3 * DEM_MAX_PLATES, 0, s, ctx->err)) return DEM_ERR_NCCL;
        CK(cudaMemcpyAsync(ctx->hub_acc, v, sizeof(v), cudaMemcpyHostToDevice, s));
    }
    launch_plate_kick(ctx->db, ctx->hub_acc, ctx->sp.h, first, s);
    ctx->launches += 2;
    return DEM_OK;
}

// Runs n Jacobi sweeps of the stage (impulses ping-pong in it_P[0/1] from it_P[0]; velocities
// from vel[cur]), replaying a captured CUDA graph when the launch configuration is unchanged
// (single context: the sweep loop has no host step between launches).  ctx->cur ends n sweeps
// later.
static dem_status item_sweeps(dem_ctx *ctx, int stage, int n, const SolveParams &sp)
{
    cudaStream_t s = ctx->s;
    const int64_t N = ctx->N;
    const int c0 = ctx->cur;
    const bool hub = mono_active(ctx);
    const bool impact = stage == 0;
    auto one = [&](int it, int a) {
        launch_sweep_items(impact, N, ctx->vel[a], ctx->ang[a], ctx->pl.rad, ctx->vel[a ^ 1], ctx->ang[a ^ 1], ctx->pl,
                           ctx->it_rec, ctx->it_P[it & 1], ctx->it_P[(it & 1) ^ 1], ctx->db, sp, s);
    };
    ctx->launches += n;
    // decomposed contexts: the loop (sweep, halo pack, grouped NCCL send/recv, unpack) is captured
    // only over a graph-safe transport without a monolithic plate (whose per-sweep allreduce
    // synchronises the host), and only on request (DEM_GRAPH_NCCL=1): NCCL inside graphs has not
    // been validated on a multi-GPU box here
    const bool capturable = !ctx->tp || (ctx->tp->graph_safe() && !hub && getenv("DEM_GRAPH_NCCL"));
    if (!capturable || n < 2 || getenv("DEM_NO_GRAPHS")) {
        for (int it = 0; it < n; it++) {
            one(it, ctx->cur);
            if (hub) TRY(plate_hub(ctx, true, ctx->it_P[it & 1], ctx->it_P[(it & 1) ^ 1], 0));
            ctx->cur ^= 1;
            TRY(halo(ctx, ctx->vel[ctx->cur], ctx->ang[ctx->cur]));
        }
        return DEM_OK;
    }
    // key: everything the captured launches bake in
    const void *ptrs[] = {ctx->vel[0], ctx->vel[1], ctx->ang[0], ctx->ang[1], ctx->pl.rad, ctx->pl.istart, ctx->pl.pin,
                          ctx->it_rec, ctx->it_P[0], ctx->it_P[1], ctx->db, ctx->it_plist, ctx->pl.item_c, ctx->geo,
                          ctx->hub_acc, ctx->hs[0], ctx->hs[1], ctx->hr[0], ctx->hr[1], ctx->send_idx[0],
                          ctx->send_idx[1], ctx->recv_idx[0], ctx->recv_idx[1]};
    const int64_t ints[] = {N, n, c0, hub ? ctx->n_it_plist : -1, ctx->n_send[0], ctx->n_send[1], ctx->n_recv[0],
                            ctx->n_recv[1]};
    std::vector<unsigned char> key(sizeof(ptrs) + sizeof(ints) + sizeof(SolveParams));
    std::memcpy(key.data(), ptrs, sizeof(ptrs));
    std::memcpy(key.data() + sizeof(ptrs), ints, sizeof(ints));
    std::memcpy(key.data() + sizeof(ptrs) + sizeof(ints), &sp, sizeof(SolveParams));
    dem_ctx::SweepGraph *cache = stage ? ctx->g_main : ctx->g_imp;
    int64_t *used = ctx->g_used[stage ? 1 : 0];
    int slot = -1, lru = 0;
    for (int q = 0; q < 4; q++) {
        if (cache[q].exec && cache[q].key == key) slot = q;
        if (used[q] < used[lru]) lru = q;
    }
    if (slot < 0) slot = lru;
    dem_ctx::SweepGraph &g = cache[slot];
    used[slot] = ++ctx->g_tick;
    if (!g.exec || g.key != key) {
        if (g.exec) { cudaGraphExecDestroy(g.exec); g.exec = nullptr; }
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        dem_status st = DEM_OK;
        for (int it = 0; it < n && st == DEM_OK; it++) {
            one(it, c0 ^ (it & 1));
            if (hub) {
                launch_plate_hub_items(ctx->n_it_plist, ctx->it_plist, ctx->pl, ctx->geo, ctx->it_rec, ctx->it_P[it & 1],
                                       ctx->it_P[(it & 1) ^ 1], ctx->hub_acc, s);
                launch_plate_kick(ctx->db, ctx->hub_acc, sp.h, 0, s);
            }
            const int a = c0 ^ (it & 1) ^ 1;   // the velocities this sweep wrote
            st = halo(ctx, ctx->vel[a], ctx->ang[a]);
        }
        const cudaError_t ce = cudaStreamEndCapture(s, &graph);
        if (st != DEM_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        CK(ce);
        CK(cudaGraphInstantiate(&g.exec, graph, 0));
        cudaGraphDestroy(graph);
        g.key = key;
    }
    CK(cudaGraphLaunch(g.exec, s));
    ctx->cur = c0 ^ (n & 1);
    return DEM_OK;
}

static dem_status step_once(dem_ctx *ctx, dem_step_report *rep)
{
    cudaStream_t s = ctx->s;
    const SolveParams &sp = ctx->sp;
    std::memset(rep, 0, sizeof(*rep));
    tstart(ctx, 0);
    if (ctx->need_rebuild) {
        TRY(agree(ctx, rebuild(ctx)));      // local failures after the band exchange (OOM): all ranks stop
        rep->rebuilt = 1;
    }
    const int64_t N = ctx->N;          // after the rebuild: the decomposition changes the local count
    tstart(ctx, 1);
    const DevBoundary hb_prev = ctx->hb;
    if (N) {
        CK(cudaMemcpyAsync(ctx->pos_prev, ctx->pos, N * sizeof(double4), cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(ctx->vel_prev, ctx->vel[ctx->cur], N * sizeof(double4), cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(ctx->ang_prev, ctx->ang[ctx->cur], N * sizeof(double4), cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaMemsetAsync(ctx->dsc, 0, sizeof(StepScalars), s));
    // narrow phase (exact predicate), compaction, incidence
    const int64_t ncand = ctx->ncand;
    launch_narrow(ncand, ctx->cand, ctx->pos, ctx->db, ctx->cflag, ctx->Pca, ctx->Pcb, ctx->dsc, s);
    scan_u32(ctx->cflag, ctx->cscan, ncand, ctx->scan_tmp, s, &ctx->launches);
    uint32_t nc = 0;
    CK(cudaMemcpyAsync(ctx->hnc, ctx->cscan + ncand, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    nc = *ctx->hnc;
    dem_status cst = DEM_OK;
    if (nc > INC_CMASK) { ctx->err = "more than 2^31 contacts on one rank"; cst = DEM_ERR_OOM; }
    else cst = ensure_contacts(ctx, std::max<int64_t>(nc, 1));
    TRY(agree(ctx, cst));
    ctx->nc = nc;
    launch_compact(ncand, ctx->cand, ctx->cflag, ctx->cscan, ctx->pos, ctx->db, sp, ctx->Pca, ctx->Pcb, ctx->cij,
                   ctx->geo, ctx->row, ctx->cdel, ctx->Pwa, ctx->Pwb, ctx->ccand, ctx->gid, ctx->dsc, s);
    launch_count_kinds(nc, OWN(ctx), ctx->cij, ctx->gid, ctx->dsc, s);
    launch_inc(N, ctx->co_start, ctx->cand, ctx->cscan, ctx->ct_start, ctx->ct_list, ctx->cflag, ctx->gid, ctx->inc_cnt,
               ctx->inc_start, ctx->inc, ctx->scan_tmp, s, &ctx->launches);
    if (ctx->sol.ordering == 0) TRY(agree(ctx, build_plan(ctx, N)));
    ctx->n_plist = 0;
    ctx->n_it_plist = 0;
    if (mono_active(ctx) && nc) {
        // monolithic plates: this step's owned plate contacts (cflag/cscan are free again)
        launch_plate_list_flags(nc, OWN(ctx), ctx->cij, ctx->cflag, s);
        scan_u32(ctx->cflag, ctx->cscan, nc, ctx->scan_tmp, s, &ctx->launches);
        uint32_t np = 0;
        CK(cudaMemcpyAsync(&np, ctx->cscan + nc, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        launch_compact_idx(nc, ctx->cflag, ctx->cscan, ctx->plist, s);
        ctx->n_plist = np;
        // ... and their items (the per-sweep increments come from the item impulses)
        const int64_t ni = ctx->n_items;
        launch_plate_items_flag(ni, OWN(ctx), ctx->pl, ctx->cij, ctx->it_flag, s);
        scan_u32(ctx->it_flag, ctx->it_scan, ni, ctx->scan_tmp, s, &ctx->launches);
        uint32_t npi = 0;
        CK(cudaMemcpyAsync(&npi, ctx->it_scan + ni, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        launch_compact_idx(ni, ctx->it_flag, ctx->it_scan, ctx->it_plist, s);
        ctx->n_it_plist = npi;
        ctx->launches += 4;
    }
    launch_prepare(N, ctx->inc_start, ctx->pos, ctx->vel[ctx->cur], ctx->ang[ctx->cur], sp.rho, s);
    TRY(halo(ctx, ctx->vel[ctx->cur], ctx->ang[ctx->cur]));      // ghosts' weights c/m, c/I from their owners
    // impact trigger
    launch_rows(nc, 0, ctx->cij, ctx->geo, ctx->cdel, ctx->row, ctx->row_imp, ctx->vel[ctx->cur], ctx->pos, ctx->db, sp, ctx->dsc, s);
    ctx->launches += 6;
    CK(cudaMemcpyAsync(ctx->hsc, ctx->dsc, sizeof(StepScalars), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    bool impact = ctx->hsc->impact != 0 && nc > 0;
    if (ctx->tp) {
        double f = impact ? 1.0 : 0.0;
        if (!ctx->tp->allreduce_f64(&f, 1, 1, s, ctx->err)) return DEM_ERR_NCCL;
        impact = f > 0.0;
    }
    tstart(ctx, 2);
    const int n_imp = ctx->sol.n_iter_impact > 0 ? ctx->sol.n_iter_impact : ctx->sol.n_iter;
    const bool gs = ctx->sol.ordering == 1;
    if (gs) {
        if (!ctx->gs_cij) {   // ordering switched on after the buffers were sized
            const int64_t cap = ctx->cap_c;
            TRY(regrow(ctx, &ctx->gs_key, cap)); TRY(regrow(ctx, &ctx->gs_col, cap)); TRY(regrow(ctx, &ctx->gs_ord, cap));
            TRY(regrow(ctx, &ctx->gs_cij, cap)); TRY(regrow(ctx, &ctx->gs_geo, cap)); TRY(regrow(ctx, &ctx->gs_row, cap));
            TRY(regrow(ctx, &ctx->gs_Pa, cap)); TRY(regrow(ctx, &ctx->gs_Pb, cap));
        }
        // colour the contact graph (priority SplitMix64(key): the oracle's greedy colouring)
        const int ncol = gs_color(nc, ctx->cij, ctx->gid, ctx->inc_start, ctx->inc, ctx->gs_key, ctx->gs_col, ctx->keys,
                                  ctx->vals, ctx->sort_tmp, ctx->gs_scr, ctx->gs_cstart, s, &ctx->launches);
        if (ncol < 0) { ctx->err = "Gauss-Seidel colouring needs more than 256 colours"; return DEM_ERR_INVALID; }
        if (nc) CK(cudaMemcpyAsync(ctx->gs_ord, ctx->vals[0], nc * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        gs_gather(nc, ctx->gs_ord, ctx->cij, ctx->geo, nullptr, nullptr, nullptr, ctx->gs_cij, ctx->gs_geo, nullptr,
                  nullptr, nullptr, s);
        ctx->launches += 1;
    }
    if (impact && gs) {
        // Newton impact stage (reading R13) in Gauss-Seidel order, in place
        gs_gather(nc, ctx->gs_ord, ctx->cij, ctx->geo, ctx->row_imp, nullptr, nullptr, nullptr, nullptr, ctx->gs_row,
                  ctx->gs_Pa, ctx->gs_Pb, s);
        for (int it = 0; it < n_imp; it++)
            gs_sweep(ctx->gs_cstart, nullptr, ctx->gs_cij, ctx->gs_geo, ctx->gs_row, ctx->gs_Pa, ctx->gs_Pb,
                     ctx->vel[ctx->cur], ctx->ang[ctx->cur], ctx->inc_start, ctx->db, sp, s, &ctx->launches);
        ctx->tm.n_sweep_launches += n_imp;
        ctx->tm.contact_sweeps += (int64_t)n_imp * nc;
        ctx->tm.particle_sweeps += (int64_t)n_imp * N;
    } else if (impact) {
        // Newton impact stage from P = 0 with Sigma = 0 (reading R13); impulses discarded
        item_pack(ctx->n_items, ctx->pl, ctx->geo, ctx->cdel, ctx->row_imp, nullptr, nullptr, ctx->it_rec, ctx->it_P[0], s);
        ctx->launches += 1;
        TRY(item_sweeps(ctx, 0, n_imp, sp));
        ctx->tm.n_sweep_launches += n_imp;
        ctx->tm.contact_sweeps += (int64_t)n_imp * nc;
        ctx->tm.particle_sweeps += (int64_t)n_imp * N;
    }
    // main stage: SPOOK rows, gravity + warm start, N_it Jacobi sweeps
    launch_rows(nc, 1, ctx->cij, ctx->geo, ctx->cdel, ctx->row, ctx->row_imp, ctx->vel[ctx->cur], ctx->pos, ctx->db, sp, ctx->dsc, s);
    launch_apply(SWEEP_MODE_APPLY, N, ctx->vel[ctx->cur], ctx->ang[ctx->cur], ctx->vel[ctx->cur ^ 1],
                 ctx->ang[ctx->cur ^ 1], ctx->inc_start, ctx->inc, ctx->geo, ctx->row, ctx->Pwa, ctx->Pwb, sp, s);
    ctx->cur ^= 1;
    ctx->launches += 2;
    TRY(halo(ctx, ctx->vel[ctx->cur], ctx->ang[ctx->cur]));
    // monolithic plates: the external impulse h F and the warm-start impulses of their contacts
    if (mono_active(ctx)) TRY(plate_hub(ctx, false, nullptr, ctx->Pwa, 1));
    tstart(ctx, 3);
    const int n_it = ctx->sol.n_iter;
    const P4 *pin_a = ctx->Pwa, *pin_b = ctx->Pwb;
    if (gs) {
        // N_it coloured Gauss-Seidel sweeps, impulses and velocities updated in place
        gs_gather(nc, ctx->gs_ord, ctx->cij, ctx->geo, ctx->row, ctx->Pwa, ctx->Pwb, nullptr, nullptr, ctx->gs_row,
                  ctx->gs_Pa, ctx->gs_Pb, s);
        for (int it = 0; it < n_it; it++)
            gs_sweep(ctx->gs_cstart, nullptr, ctx->gs_cij, ctx->gs_geo, ctx->gs_row, ctx->gs_Pa, ctx->gs_Pb,
                     ctx->vel[ctx->cur], ctx->ang[ctx->cur], ctx->inc_start, ctx->db, sp, s, &ctx->launches);
        gs_scatter(nc, ctx->gs_ord, ctx->gs_Pa, ctx->gs_Pb, ctx->Pa[0], ctx->Pb[0], s);
        ctx->launches += 3;
        pin_a = ctx->Pa[0];
        pin_b = ctx->Pb[0];
    } else if (n_it > 0) {
        // N_it Jacobi sweeps from the warm start, then the final impulses back to the contacts
        item_pack(ctx->n_items, ctx->pl, ctx->geo, ctx->cdel, ctx->row, ctx->Pwa, ctx->Pwb, ctx->it_rec, ctx->it_P[0], s);
        TRY(item_sweeps(ctx, 1, n_it, sp));
        item_unpack(ctx->n_items, ctx->pl, ctx->it_rec, ctx->it_P[n_it & 1], ctx->Pa[0], ctx->Pb[0], s);
        ctx->launches += 2;
        pin_a = ctx->Pa[0];
        pin_b = ctx->Pb[0];
    }
    ctx->tm.n_sweep_launches += n_it;
    ctx->tm.contact_sweeps += (int64_t)n_it * nc;
    ctx->tm.particle_sweeps += (int64_t)n_it * N;
    tstart(ctx, 4);
    ctx->Pfa = (P4 *)pin_a;
    ctx->Pfb = (P4 *)pin_b;
    launch_residuals(nc, OWN(ctx), ctx->cij, ctx->geo, ctx->row, ctx->vel[ctx->cur], ctx->Pfa, ctx->Pfb, ctx->db, sp,
                     ctx->dsc, s);
    // integrate, plates and walls
    launch_integrate(N, OWN(ctx), ctx->pos, ctx->vel[ctx->cur], ctx->ang[ctx->cur], ctx->xref, sp.h, sp.rho, ctx->ke_part,
                     ctx->dsc, s);
    launch_plate_sum(nc, OWN(ctx), ctx->cij, ctx->geo, ctx->Pfa, ctx->pacc, ctx->pcount, s);
    if (ctx->tp) {
        // plate and wall reactions: exact int64 sums over the ranks (each contact counted by its owner)
        unsigned long long acc[3 * NB_SLOTS];
        unsigned int pc[NB_SLOTS];
        CK(cudaMemcpyAsync(acc, ctx->pacc, sizeof(acc), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(pc, ctx->pcount, sizeof(pc), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        long long v[4 * NB_SLOTS];
        for (int q = 0; q < 3 * NB_SLOTS; q++) v[q] = (long long)acc[q];
        for (int q = 0; q < NB_SLOTS; q++) v[3 * NB_SLOTS + q] = pc[q];
        if (!ctx->tp->allreduce_i64(v, 4 * NB_SLOTS, 0, s, ctx->err)) return DEM_ERR_NCCL;
        for (int q = 0; q < 3 * NB_SLOTS; q++) acc[q] = (unsigned long long)v[q];
        for (int q = 0; q < NB_SLOTS; q++) pc[q] = (unsigned int)v[3 * NB_SLOTS + q];
        CK(cudaMemcpyAsync(ctx->pacc, acc, sizeof(acc), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->pcount, pc, sizeof(pc), cudaMemcpyHostToDevice, s));
    }
    launch_boundary(ctx->db, ctx->pacc, ctx->pcount, sp.h, ctx->dsc, s);
    ctx->launches += (N ? 2 : 0) + (nc ? 2 : 1);
    CK(cudaMemcpyAsync(ctx->hsc, ctx->dsc, sizeof(StepScalars), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&ctx->hb, ctx->db, sizeof(DevBoundary), cudaMemcpyDeviceToHost, s));
    tstart(ctx, 5);
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    StepScalars sc = *ctx->hsc;
    if (ctx->tp) {
        // global report and decisions: every rank takes the same rollback / rebuild branch
        double mx[5], sm[5];
        std::memcpy(&mx[0], &sc.max_disp_bits, 8);
        std::memcpy(&mx[1], &sc.max_v_bits, 8);
        mx[2] = sc.nan_flag ? 1.0 : 0.0;
        std::memcpy(&mx[3], &sc.max_res_bits, 8);
        std::memcpy(&mx[4], &sc.max_cone_bits, 8);
        sm[0] = sc.ke; sm[1] = sc.n_pp; sm[2] = sc.n_wall; sm[3] = sc.n_plate; sm[4] = sc.n_degenerate;
        if (!ctx->tp->allreduce_f64(mx, 5, 1, s, ctx->err) || !ctx->tp->allreduce_f64(sm, 5, 0, s, ctx->err))
            return DEM_ERR_NCCL;
        std::memcpy(&sc.max_disp_bits, &mx[0], 8);
        std::memcpy(&sc.max_v_bits, &mx[1], 8);
        std::memcpy(&sc.max_res_bits, &mx[3], 8);
        std::memcpy(&sc.max_cone_bits, &mx[4], 8);
        sc.nan_flag = mx[2] > 0.0 ? 1u : 0u;
        sc.ke = sm[0];
        sc.n_pp = (unsigned)sm[1]; sc.n_wall = (unsigned)sm[2]; sc.n_plate = (unsigned)sm[3]; sc.n_degenerate = (unsigned)sm[4];
    }
    if (sc.nan_flag) {
        // name the first offending contact (smallest key) or particle, over all ranks
        unsigned long long bad[2] = {~0ull, ~0ull};
        if (!ctx->dscr_bad) TRY(A(ctx, &ctx->dscr_bad, 2));
        launch_first_bad(nc, N, OWN(ctx), ctx->cij, ctx->gid, ctx->Pfa, ctx->Pfb, ctx->pos, ctx->vel[ctx->cur],
                         ctx->ang[ctx->cur], ctx->dscr_bad, s);
        CK(cudaMemcpyAsync(bad, ctx->dscr_bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (ctx->tp) {
            // global minimum of each 64-bit key: high words first, then the low words of the ranks
            // holding the minimal high word (max of negatives, exact in int64)
            for (int q = 0; q < 2; q++) {
                long long hi = -(long long)(bad[q] >> 32);
                if (!ctx->tp->allreduce_i64(&hi, 1, 1, s, ctx->err)) return DEM_ERR_NCCL;
                const unsigned long long ghi = (unsigned long long)(-hi);
                long long lo = (bad[q] >> 32) == ghi ? -(long long)(bad[q] & 0xFFFFFFFFull) : -(1ll << 32);
                if (!ctx->tp->allreduce_i64(&lo, 1, 1, s, ctx->err)) return DEM_ERR_NCCL;
                bad[q] = (ghi << 32) | (unsigned long long)(-lo);
            }
        }
        std::string where = "";
        if (bad[0] != ~0ull)
            where = " at contact key " + std::to_string(bad[0]) + " (gid " + std::to_string(bad[0] >> 32) + ", partner " +
                    std::to_string(bad[0] & 0xFFFFFFFFull) + ")";
        else if (bad[1] != ~0ull)
            where = " at particle gid " + std::to_string(bad[1] >> 32);
        // atomic step: restore the state of the step start
        if (N) {
            CK(cudaMemcpyAsync(ctx->pos, ctx->pos_prev, N * sizeof(double4), cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(ctx->vel[ctx->cur], ctx->vel_prev, N * sizeof(double4), cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(ctx->ang[ctx->cur], ctx->ang_prev, N * sizeof(double4), cudaMemcpyDeviceToDevice, s));
        }
        ctx->hb = hb_prev;
        TRY(upload_boundary(ctx));
        CK(cudaStreamSynchronize(s));
        ctx->have_step = false;
        ctx->err = "step " + std::to_string(ctx->step + 1) + " diverged (NaN/Inf)" + where + "; state rolled back";
        return DEM_ERR_DIVERGED;
    }
    launch_scatter_P(nc, ctx->ccand, ctx->Pfa, ctx->Pfb, ctx->Pca, ctx->Pcb, s);
    ctx->launches += nc ? 1 : 0;
    TRY(sync_check(ctx, "step end"));
    if (ctx->timing) {
        ctx->tm.ms_rebuild += telapsed(ctx, 0, 1);
        ctx->tm.ms_detect += telapsed(ctx, 1, 2);
        ctx->tm.ms_sweeps += telapsed(ctx, 2, 4) ;
        ctx->tm.ms_integrate += telapsed(ctx, 4, 5);
        ctx->tm.ms_total += telapsed(ctx, 0, 5);
    }
    double maxd, maxv;
    {
        unsigned long long b = sc.max_disp_bits;
        std::memcpy(&maxd, &b, 8);
        b = sc.max_v_bits;
        std::memcpy(&maxv, &b, 8);
    }
    ctx->step++;
    rep->step = ctx->step;
    rep->time = ctx->hb.time;
    rep->n_contacts = ctx->tp ? (int64_t)sc.n_pp + sc.n_wall + sc.n_plate : (int64_t)nc;
    rep->n_pp = sc.n_pp;
    rep->n_wall = sc.n_wall;
    rep->n_plate = sc.n_plate;
    rep->n_degenerate = sc.n_degenerate;
    rep->n_candidates = ncand;
    rep->impact_fired = impact ? 1 : 0;
    rep->ke = sc.ke;
    rep->max_v = maxv;
    rep->max_disp = maxd;
    std::memcpy(&rep->max_normal_residual, &sc.max_res_bits, 8);
    std::memcpy(&rep->max_cone_excess, &sc.max_cone_bits, 8);
    rep->n_iter = n_it;
    rep->n_colors = gs ? (int32_t)ctx->gs_cstart.size() - 1 : 0;
    rep->n_iter_impact = impact ? n_imp : 0;
    const double skin = ctx->grid.skin;
    ctx->need_rebuild = (2.0 * maxd >= 0.9 * skin) || (maxd + sc.bnd_disp >= 0.9 * skin);
    ctx->have_step = true;
    ctx->last = *rep;
    return DEM_OK;
}

// ------------------------------------------------------------------ state loading
// host copies of a particle set being loaded, validated before the context is touched
struct HostSet { std::vector<double> r, x; std::vector<uint32_t> g, gs; };
static dem_status validate_particles(dem_ctx *ctx, int64_t n, const double *pos, const double *rad, const uint32_t *gid,
                                     int on_device, bool check_slab, HostSet &h)
{
    h.r.resize(n); h.x.resize(3 * n); h.g.resize(n);
    cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
    if (n) {
        CK(cudaMemcpy(h.r.data(), rad, n * 8, kind));
        CK(cudaMemcpy(h.x.data(), pos, 3 * n * 8, kind));
        if (gid) CK(cudaMemcpy(h.g.data(), gid, n * 4, kind));
        else for (int64_t i = 0; i < n; i++) h.g[i] = (uint32_t)i;
    }
    for (int64_t i = 0; i < n; i++) {
        if (!(h.r[i] > 0) || !std::isfinite(h.r[i])) { ctx->err = "radius must be positive and finite"; return DEM_ERR_INVALID; }
        for (int k = 0; k < 3; k++) if (!std::isfinite(h.x[3 * i + k])) { ctx->err = "non-finite position"; return DEM_ERR_INVALID; }
        if (h.g[i] >= PLATE_KEY_BASE) { ctx->err = "gid must be < 2^32-4096"; return DEM_ERR_INVALID; }
        if (check_slab && ctx->tp && !((ctx->rank == 0 || h.x[3 * i] >= ctx->slab_lo) && (ctx->rank == ctx->G - 1 || h.x[3 * i] < ctx->slab_hi))) {
            ctx->err = "particle outside this rank's slab [slab_lo, slab_hi)";
            return DEM_ERR_INVALID;
        }
    }
    h.gs = h.g;
    std::sort(h.gs.begin(), h.gs.end());
    for (int64_t i = 1; i < n; i++) if (h.gs[i] == h.gs[i - 1]) { ctx->err = "duplicate gid"; return DEM_ERR_INVALID; }
    return DEM_OK;
}

// loads a validated set (first: new particle arrays; else: same count as the context's)
static dem_status commit_particles(dem_ctx *ctx, int64_t n, const HostSet &h, const double *pos, const double *rad,
                                   const double *vel, const double *ang, int on_device, bool first)
{
    const std::vector<double> &r = h.r;
    const std::vector<uint32_t> &g = h.g, &gs = h.gs;
    if (first) {
        TRY(alloc_particles(ctx, n));     // counts are set once the arrays exist (an OOM leaves them as they were)
        ctx->N = n;
        ctx->N_own = n;
    } else if (n != ctx->N) {
        ctx->err = "set_state: particle count differs from create";
        return DEM_ERR_INVALID;
    }
    TRY(setup_levels(ctx, r));
    // stage host copies into device buffers, then convert to the internal layout
    double *dx = nullptr, *dr = nullptr, *dv = nullptr, *dw = nullptr;
    uint32_t *dg = nullptr;
    if (n) {
        TRY(A(ctx, &dx, 3 * n)); TRY(A(ctx, &dr, n)); TRY(A(ctx, &dg, n));
        if (vel) TRY(A(ctx, &dv, 3 * n));
        if (ang) TRY(A(ctx, &dw, 3 * n));
        cudaMemcpyKind k2 = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        CK(cudaMemcpyAsync(dx, pos, 3 * n * 8, k2, ctx->s));
        CK(cudaMemcpyAsync(dr, rad, n * 8, k2, ctx->s));
        CK(cudaMemcpyAsync(dg, g.data(), n * 4, cudaMemcpyHostToDevice, ctx->s));
        if (vel) CK(cudaMemcpyAsync(dv, vel, 3 * n * 8, k2, ctx->s));
        if (ang) CK(cudaMemcpyAsync(dw, ang, 3 * n * 8, k2, ctx->s));
        ctx->cur = 0;
        launch_load_state(n, dx, dr, dv, dw, dg, ctx->pos, ctx->vel[0], ctx->ang[0], ctx->gid, ctx->s);
        ctx->launches++;
        CK(cudaMemcpyAsync(ctx->gid_sorted, gs.data(), n * 4, cudaMemcpyHostToDevice, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        dfree(ctx, dx); dfree(ctx, dr); dfree(ctx, dg); dfree(ctx, dv); dfree(ctx, dw);
    }
    ctx->need_rebuild = true;
    ctx->have_step = false;
    return DEM_OK;
}

static dem_status load_particles(dem_ctx *ctx, int64_t n, const double *pos, const double *rad, const double *vel,
                                 const double *ang, const uint32_t *gid, int on_device, bool first, bool check_slab = true)
{
    HostSet h;
    TRY(validate_particles(ctx, n, pos, rad, gid, on_device, check_slab, h));
    return commit_particles(ctx, n, h, pos, rad, vel, ang, on_device, first);
}

// ------------------------------------------------------------------ C-ABI
extern "C" {

dem_status dem_create_bed(const dem_bed_desc *desc, const dem_dist_desc *dist, dem_ctx **out)
{
    if (!desc || !out) { g_create_err = "null descriptor"; return DEM_ERR_INVALID; }
    *out = nullptr;
    if (desc->struct_size != sizeof(dem_bed_desc)) { g_create_err = "dem_bed_desc struct_size mismatch"; return DEM_ERR_INVALID; }
    if (!valid_material(desc->mat)) { g_create_err = "invalid material"; return DEM_ERR_INVALID; }
    const dem_solver &so = desc->solver;
    if (!(so.dt > 0) || so.n_iter < 1 || !(so.ordering == 0 || so.ordering == 1) || !(so.reduction == 0 || so.reduction == 1) ||
        !(so.plate_coupling == 0 || so.plate_coupling == 1) || (so.plate_coupling == 1 && so.ordering == 1) ||
        !(so.hertz_exp == 1.25 || so.hertz_exp == 1.0) ||
        (so.hertz_exp == 1.0 && !(so.k_lin > 0)) || so.damping_steps < 0) {
        g_create_err = "invalid solver settings (dt > 0, n_iter >= 1, hertz_exp 1.25 or 1 with k_lin > 0)";
        return DEM_ERR_INVALID;
    }
    for (int k = 0; k < 3; k++)
        if (!(desc->box.lo[k] < desc->box.hi[k])) { g_create_err = "box lo must be < hi"; return DEM_ERR_INVALID; }
    if (desc->source != 0 && desc->source != 1) { g_create_err = "source must be 0 (particles) or 1 (generator)"; return DEM_ERR_INVALID; }
    if (desc->source == 0 && (desc->parts.n < 0 || (desc->parts.n > 0 && (!desc->parts.pos || !desc->parts.radius)))) {
        g_create_err = "particle arrays missing";
        return DEM_ERR_INVALID;
    }
    if (desc->parts.n >= (int64_t)0x7FFFFFFF) { g_create_err = "too many particles for one context"; return DEM_ERR_INVALID; }
    // decomposition active: world_size > 1, or any explicit transport (one rank over NCCL/loopback
    // runs the same decomposed code path with no neighbours: the transport self-test)
    const bool decomposed = dist && (dist->world_size > 1 || dist->nccl_unique_id || dist->loopback);
    if (decomposed) {
        if (dist->world_size < 1 || dist->rank < 0 || dist->rank >= dist->world_size || !(dist->slab_lo < dist->slab_hi) ||
            (dist->transport != 0 && dist->transport != 1) || (dist->transport == 1 && !dist->loopback)) {
            g_create_err = "invalid decomposition (rank, slab_lo < slab_hi, transport 0 NCCL | 1 loopback)";
            return DEM_ERR_INVALID;
        }
    }
    dem_ctx *ctx = new dem_ctx();
    ctx->mat = desc->mat;
    ctx->sol = desc->solver;
    ctx->box = desc->box;
    if (dist && dist->cuda_stream) ctx->s = (cudaStream_t)dist->cuda_stream;
    else {
        if (cudaStreamCreateWithFlags(&ctx->s, cudaStreamNonBlocking) != cudaSuccess) {
            g_create_err = "cudaStreamCreate failed (no CUDA device?)";
            delete ctx;
            return DEM_ERR_CUDA;
        }
        ctx->own_stream = true;
    }
    if (dist && dist->alloc && dist->free) { ctx->ualloc = dist->alloc; ctx->ufree = dist->free; ctx->actx = dist->alloc_ctx; }
    if (decomposed) {
        ctx->G = dist->world_size;
        ctx->rank = dist->rank;
        ctx->slab_lo = dist->slab_lo;
        ctx->slab_hi = dist->slab_hi;
        std::string err;
        ctx->tp = dist->transport == 1 ? make_loop_transport(ctx->rank, (LoopGroup *)dist->loopback, err)
                                       : make_nccl_transport(ctx->rank, ctx->G, dist->nccl_unique_id, err);
        if (!ctx->tp) {
            g_create_err = err;
            dem_destroy(ctx);
            return DEM_ERR_NCCL;
        }
    }
    setup_solve_params(ctx);
    setup_walls(ctx);
    for (int e = 0; e < 8; e++) cudaEventCreate(&ctx->ev[e]);
    if (cudaMallocHost(&ctx->hsc, sizeof(StepScalars)) != cudaSuccess ||
        cudaMallocHost(&ctx->hnc, sizeof(uint32_t)) != cudaSuccess) {
        g_create_err = "cudaMallocHost failed";
        dem_destroy(ctx);
        return DEM_ERR_CUDA;
    }
    const dem_particles &p = desc->parts;
    dem_status st;
    if (desc->source == 1) {
        // on-device generator: this rank's sites (outer slabs open), then the standard load
        const double lo = (!ctx->tp || ctx->rank == 0) ? -INFINITY : ctx->slab_lo;
        const double hi = (!ctx->tp || ctx->rank == ctx->G - 1) ? INFINITY : ctx->slab_hi;
        double *gx = nullptr, *gr = nullptr;
        uint32_t *gg = nullptr;
        int64_t gn = 0;
        std::string gerr;
        if (!generate_bed(desc->gen, desc->box, lo, hi, ctx_alloc, ctx, ctx->s, &gx, &gr, &gg, &gn, gerr)) {
            ctx->err = gerr;
            st = DEM_ERR_INVALID;
        } else {
            // jittered sites may sit a hair outside the slab: the first rebuild assigns them
            st = load_particles(ctx, gn, gx, gr, nullptr, nullptr, gg, 1, true, false);
        }
        for (void *q : {(void *)gx, (void *)gr, (void *)gg}) dfree(ctx, q);
    } else {
        st = load_particles(ctx, p.n, p.pos, p.radius, p.vel, p.angvel, p.gid, p.on_device, true);
    }
    if (st == DEM_OK) st = upload_boundary(ctx);
    if (st == DEM_OK) st = rebuild(ctx);
    if (st != DEM_OK) {
        g_create_err = ctx->err;
        dem_destroy(ctx);
        return st;
    }
    *out = ctx;
    return DEM_OK;
}

dem_status dem_step(dem_ctx *ctx, int32_t n_steps, dem_step_report *last)
{
    if (!ctx) return DEM_ERR_INVALID;
    if (n_steps < 1) { ctx->err = "n_steps must be >= 1"; return DEM_ERR_INVALID; }
    dem_step_report rep{};
    for (int32_t k = 0; k < n_steps; k++) TRY(step_once(ctx, &rep));
    if (last) *last = rep;
    return DEM_OK;
}

static bool valid_solver(const dem_solver &so)
{
    return (so.ordering == 0 || so.ordering == 1) && (so.reduction == 0 || so.reduction == 1) &&
           (so.plate_coupling == 0 || (so.plate_coupling == 1 && so.ordering == 0)) && so.dt > 0 &&
           so.n_iter >= 1 && (so.hertz_exp == 1.25 || so.hertz_exp == 1.0) &&
           !(so.hertz_exp == 1.0 && !(so.k_lin > 0)) && so.damping_steps >= 0;
}

dem_status dem_set_solver(dem_ctx *ctx, const dem_solver *so)
{
    if (!ctx || !so) return DEM_ERR_INVALID;
    if (!valid_solver(*so)) { ctx->err = "invalid solver settings"; return DEM_ERR_INVALID; }
    if (ctx->tp && so->ordering == 1) { ctx->err = "Gauss-Seidel ordering needs a single undecomposed context"; return DEM_ERR_INVALID; }
    const double skin = ctx->grid.skin;
    ctx->sol = *so;
    setup_solve_params(ctx);
    ctx->grid.skin = skin;
    return upload_boundary(ctx);
}

dem_status dem_get_state(dem_ctx *ctx, dem_state_view *v)
{
    if (!ctx || !v) return DEM_ERR_INVALID;
    if (v->n < ctx->N_own) { ctx->err = "state view too small"; v->n = ctx->N_own; return DEM_ERR_INVALID; }
    const int64_t N = ctx->N_own;        // owned particles (all of them with world_size 1)
    v->n = N;
    if (!N) return DEM_OK;
    cudaStream_t s = ctx->s;
    if (v->on_device) {
        launch_to_gid_order(ctx->N, N, OWN(ctx), ctx->gid, ctx->gid_sorted, ctx->pos, ctx->vel[ctx->cur], ctx->ang[ctx->cur], v->pos,
                            v->vel, v->angvel, v->radius, v->gid, s);
        ctx->launches++;
        CK(cudaStreamSynchronize(s));
        return DEM_OK;
    }
    double *d = nullptr;
    uint32_t *dg = nullptr;
    TRY(A(ctx, &d, 10 * N));
    TRY(A(ctx, &dg, N));
    launch_to_gid_order(ctx->N, N, OWN(ctx), ctx->gid, ctx->gid_sorted, ctx->pos, ctx->vel[ctx->cur], ctx->ang[ctx->cur], d, d + 3 * N,
                        d + 6 * N, d + 9 * N, dg, s);
    ctx->launches++;
    if (v->pos) CK(cudaMemcpyAsync(v->pos, d, 3 * N * 8, cudaMemcpyDeviceToHost, s));
    if (v->vel) CK(cudaMemcpyAsync(v->vel, d + 3 * N, 3 * N * 8, cudaMemcpyDeviceToHost, s));
    if (v->angvel) CK(cudaMemcpyAsync(v->angvel, d + 6 * N, 3 * N * 8, cudaMemcpyDeviceToHost, s));
    if (v->radius) CK(cudaMemcpyAsync(v->radius, d + 9 * N, N * 8, cudaMemcpyDeviceToHost, s));
    if (v->gid) CK(cudaMemcpyAsync(v->gid, dg, N * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(ctx, d);
    dfree(ctx, dg);
    return DEM_OK;
}

dem_status dem_set_state(dem_ctx *ctx, const dem_state_view *st, const dem_contact_view *hist)
{
    if (!ctx || !st) return DEM_ERR_INVALID;
    if (ctx->tp) { ctx->err = "dem_set_state needs world_size 1"; return DEM_ERR_INVALID; }
    if (st->n != ctx->N || (st->n && (!st->pos || !st->radius))) { ctx->err = "set_state: bad view"; return DEM_ERR_INVALID; }
    // history: sorted by key on the host, uploaded for the next rebuild's sorted-key lookup
    std::vector<uint64_t> hk;
    std::vector<P4> ha, hbv;
    if (hist && hist->n > 0) {
        const int64_t n = hist->n;
        std::vector<uint64_t> k(n);
        std::vector<double> P(7 * n);
        cudaMemcpyKind kind = hist->on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
        CK(cudaMemcpy(k.data(), hist->key, n * 8, kind));
        CK(cudaMemcpy(P.data(), hist->P, 7 * n * 8, kind));
        std::vector<int64_t> ord(n);
        for (int64_t i = 0; i < n; i++) ord[i] = i;
        std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return k[a] < k[b]; });
        for (int64_t t = 0; t < n; t++) {
            const int64_t i = ord[t];
            if (t && k[i] == hk.back()) { ctx->err = "set_state: duplicate history key"; return DEM_ERR_INVALID; }
            hk.push_back(k[i]);
            ha.push_back(mkP4(P[7 * i], P[7 * i + 1], P[7 * i + 2], P[7 * i + 3]));
            hbv.push_back(mkP4(P[7 * i + 4], P[7 * i + 5], P[7 * i + 6], 0));
        }
    }
    TRY(load_particles(ctx, st->n, st->pos, st->radius, st->vel, st->angvel, st->gid, st->on_device, false));
    const int64_t nh = (int64_t)hk.size();
    if (nh > ctx->cap_h) {
        int64_t cap = nh + 1024;
        TRY(regrow(ctx, &ctx->hkey, cap)); TRY(regrow(ctx, &ctx->hPa, cap)); TRY(regrow(ctx, &ctx->hPb, cap));
        TRY(regrow(ctx, &ctx->hauth, cap));
        ctx->cap_h = cap;
    }
    if (nh) {
        CK(cudaMemcpyAsync(ctx->hkey, hk.data(), nh * 8, cudaMemcpyHostToDevice, ctx->s));
        CK(cudaMemcpyAsync(ctx->hPa, ha.data(), nh * sizeof(P4), cudaMemcpyHostToDevice, ctx->s));
        CK(cudaMemcpyAsync(ctx->hPb, hbv.data(), nh * sizeof(P4), cudaMemcpyHostToDevice, ctx->s));
    }
    ctx->nh = nh;
    ctx->hist_pending = true;
    // the caller's history is global (every rank gets all of it): nothing to hand over
    if (nh && ctx->hauth) CK(cudaMemsetAsync(ctx->hauth, 0, nh, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return rebuild(ctx);
}

dem_status dem_get_contacts(dem_ctx *ctx, dem_contact_view *v)
{
    if (!ctx || !v) return DEM_ERR_INVALID;
    if (!ctx->have_step) { ctx->err = "no step taken yet"; return DEM_ERR_STATE; }
    const int64_t ncl = ctx->nc;
    cudaStream_t s = ctx->s;
    // contacts this rank reports (all with world_size 1): owner of the smaller gid / the particle
    unsigned int *dcnt = nullptr, hcnt = 0;
    TRY(A(ctx, &dcnt, 1));
    CK(cudaMemsetAsync(dcnt, 0, 4, s));
    launch_contact_keys(ncl, OWN(ctx), ctx->cij, ctx->gid, ctx->keys[0], ctx->vals[0], dcnt, s);
    CK(cudaMemcpyAsync(&hcnt, dcnt, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(ctx, dcnt);
    const int64_t nc = hcnt;
    if (v->n < nc) { v->n = nc; ctx->err = "contact view too small"; return DEM_ERR_INVALID; }
    v->n = nc;
    if (!nc) return DEM_OK;
    radix_sort_u64(ctx->keys, ctx->vals, ncl, 64, ctx->sort_tmp, s, &ctx->launches);
    double *d = nullptr;
    TRY(A(ctx, &d, 11 * nc));
    launch_contact_out(nc, ctx->vals[0], ctx->cij, ctx->gid, ctx->geo, ctx->cdel, ctx->Pfa, ctx->Pfb, d, d + 3 * nc, d + 4 * nc, s);
    ctx->launches += 2;
    cudaMemcpyKind k = v->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (v->key) CK(cudaMemcpyAsync(v->key, ctx->keys[0], nc * 8, k, s));
    if (v->normal) CK(cudaMemcpyAsync(v->normal, d, 3 * nc * 8, k, s));
    if (v->delta) CK(cudaMemcpyAsync(v->delta, d + 3 * nc, nc * 8, k, s));
    if (v->P) CK(cudaMemcpyAsync(v->P, d + 4 * nc, 7 * nc * 8, k, s));
    CK(cudaStreamSynchronize(s));
    dfree(ctx, d);
    return DEM_OK;
}

dem_status dem_get_forces(dem_ctx *ctx, double *F, double *T, int32_t on_device)
{
    if (!ctx) return DEM_ERR_INVALID;
    if (!ctx->have_step) { ctx->err = "no step taken yet"; return DEM_ERR_STATE; }
    const int64_t N = ctx->N, Nown = ctx->N_own;
    if (!N) return DEM_OK;
    cudaStream_t s = ctx->s;
    launch_apply(SWEEP_MODE_FORCES, N, ctx->vel[ctx->cur], ctx->ang[ctx->cur], ctx->vel_prev, ctx->ang_prev, ctx->inc_start,
                 ctx->inc, ctx->geo, ctx->row, ctx->Pfa, ctx->Pfb, ctx->sp, s);
    double *d = nullptr;
    TRY(A(ctx, &d, 6 * N));
    launch_to_gid_order(N, Nown, OWN(ctx), ctx->gid, ctx->gid_sorted, ctx->vel_prev, ctx->ang_prev, nullptr, d, d + 3 * Nown, nullptr, nullptr,
                        nullptr, s);
    ctx->launches += 2;
    cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (F) CK(cudaMemcpyAsync(F, d, 3 * Nown * 8, k, s));
    if (T) CK(cudaMemcpyAsync(T, d + 3 * Nown, 3 * Nown * 8, k, s));
    CK(cudaStreamSynchronize(s));
    dfree(ctx, d);
    return DEM_OK;
}

dem_status dem_add_plate(dem_ctx *ctx, const dem_plate_desc *d, const double pos[3], int32_t *plate_id)
{
    if (!ctx || !d || !pos) return DEM_ERR_INVALID;
    DevBoundary &b = ctx->hb;
    if (b.n_plates >= DEM_MAX_PLATES) { ctx->err = "too many plates (max 8)"; return DEM_ERR_INVALID; }
    if (d->n_boxes < 1 || d->n_boxes > DEM_MAX_BOXES || !d->lo || !d->hi || !(d->mass > 0) || d->mu_t < 0 || d->mu_r < 0) {
        ctx->err = "invalid plate descriptor";
        return DEM_ERR_INVALID;
    }
    for (int q = 0; q < d->n_boxes; q++)
        for (int k = 0; k < 3; k++)
            if (!(d->lo[3 * q + k] < d->hi[3 * q + k])) { ctx->err = "plate box lo must be < hi"; return DEM_ERR_INVALID; }
    const int p = b.n_plates;
    b.nbox[p] = d->n_boxes;
    for (int q = 0; q < d->n_boxes; q++)
        for (int k = 0; k < 3; k++) { b.lo[p][q][k] = d->lo[3 * q + k]; b.hi[p][q][k] = d->hi[3 * q + k]; }
    for (int k = 0; k < 3; k++) {
        b.ppos[p][k] = pos[k];
        b.ppos_ref[p][k] = pos[k];
        b.pvel[p][k] = 0;
        b.mode[p][k] = DEM_AXIS_LOCKED;
        b.target[p][k] = 0;
        b.ramp[p][k] = 0;
        b.t0[p][k] = 0;
        b.pforce[p][k] = 0;
        b.pmotor[p][k] = 0;
        b.plimit[p][k] = 0;
        b.pfmin[p][k] = -INFINITY;
        b.pfmax[p][k] = INFINITY;
    }
    b.pmass[p] = d->mass;
    b.pmu_t[p] = d->mu_t;
    b.pmu_r[p] = d->mu_r;
    b.pcount[p] = 0;
    b.n_plates = p + 1;
    if (plate_id) *plate_id = p;
    TRY(upload_boundary(ctx));
    ctx->need_rebuild = true;
    return DEM_OK;
}

dem_status dem_drive_plate(dem_ctx *ctx, int32_t plate, int32_t axis, int32_t mode, double target, double ramp_time,
                           double f_min, double f_max)
{
    if (!ctx) return DEM_ERR_INVALID;
    DevBoundary &b = ctx->hb;
    if (plate < 0 || plate >= b.n_plates || axis < 0 || axis > 2 || mode < 0 || mode > 2 || !std::isfinite(target) ||
        !(ramp_time >= 0) || std::isnan(f_min) || std::isnan(f_max) || !(f_min <= f_max)) {
        ctx->err = "invalid plate drive";
        return DEM_ERR_INVALID;
    }
    b.mode[plate][axis] = mode;
    b.target[plate][axis] = target;
    b.ramp[plate][axis] = ramp_time;
    b.t0[plate][axis] = b.time;
    b.plimit[plate][axis] = mode == DEM_AXIS_VELOCITY && (f_min > -INFINITY || f_max < INFINITY);
    b.pfmin[plate][axis] = f_min;
    b.pfmax[plate][axis] = f_max;
    // an unlimited motor takes its speed at once (from rest if ramped); a force-limited one keeps
    // the current velocity and is accelerated by its motor from the next step on
    if (mode == DEM_AXIS_LOCKED) b.pvel[plate][axis] = 0;
    else if (mode == DEM_AXIS_VELOCITY && !b.plimit[plate][axis]) b.pvel[plate][axis] = ramp_time > 0 ? 0.0 : target;
    return upload_boundary(ctx);
}

dem_status dem_get_plate(dem_ctx *ctx, int32_t plate, dem_plate_state *o)
{
    if (!ctx || !o) return DEM_ERR_INVALID;
    const DevBoundary &b = ctx->hb;
    if (plate < 0 || plate >= b.n_plates) { ctx->err = "no such plate"; return DEM_ERR_INVALID; }
    for (int k = 0; k < 3; k++) { o->pos[k] = b.ppos[plate][k]; o->vel[k] = b.pvel[plate][k]; o->force[k] = b.pforce[plate][k];
                                    o->motor_force[k] = b.pmotor[plate][k]; }
    o->n_contacts = b.pcount[plate];
    return DEM_OK;
}

dem_status dem_get_wall(dem_ctx *ctx, int32_t wall, dem_wall_state *o)
{
    if (!ctx || !o) return DEM_ERR_INVALID;
    const DevBoundary &b = ctx->hb;
    if (wall < 0 || wall > 5 || !b.wpresent[wall]) { ctx->err = "no such wall"; return DEM_ERR_INVALID; }
    for (int k = 0; k < 3; k++) { o->point[k] = b.wp[wall][k]; o->normal[k] = b.wn[wall][k]; o->force[k] = b.wforce[wall][k]; }
    o->velocity = b.wvel[wall];
    o->n_contacts = b.wcount[wall];
    return DEM_OK;
}

dem_status dem_drive_wall(dem_ctx *ctx, int32_t wall, double v)
{
    if (!ctx) return DEM_ERR_INVALID;
    if (wall < 0 || wall > 5 || !ctx->hb.wpresent[wall] || !std::isfinite(v)) { ctx->err = "invalid wall"; return DEM_ERR_INVALID; }
    ctx->hb.wvel[wall] = v;
    return upload_boundary(ctx);
}

dem_status dem_set_timing(dem_ctx *ctx, int32_t enable)
{
    if (!ctx) return DEM_ERR_INVALID;
    ctx->timing = enable != 0;
    return DEM_OK;
}
dem_status dem_get_timing(dem_ctx *ctx, dem_timing *o)
{
    if (!ctx || !o) return DEM_ERR_INVALID;
    *o = ctx->tm;
    o->n_kernel_launches = ctx->launches;
    return DEM_OK;
}
dem_status dem_reset_timing(dem_ctx *ctx)
{
    if (!ctx) return DEM_ERR_INVALID;
    ctx->tm = dem_timing{};
    ctx->launches = 0;
    return DEM_OK;
}

// Diagnostic: time n Jacobi sweeps of the shipped sweep kernel (variant 0, the only one) on the
// last step's contact set: inputs are the current velocities and the last step's final
// impulses with the main-stage rows.  Leaves the particle state and the contact getters
// untouched (the sweeps write scratch buffers).  *max_dv_rel is 0 (kept for the ABI).
dem_status dem_bench_sweeps(dem_ctx *ctx, int32_t variant, int32_t n, double *ms_per_sweep, double *max_dv_rel)
{
    if (!ctx || n < 1) return DEM_ERR_INVALID;
    if (!ctx->have_step) { ctx->err = "no step taken yet"; return DEM_ERR_STATE; }
    if (ctx->tp) { ctx->err = "dem_bench_sweeps needs world_size 1"; return DEM_ERR_INVALID; }
    if (variant != 0) { ctx->err = "dem_bench_sweeps: only variant 0 (the shipped sweep) exists"; return DEM_ERR_INVALID; }
    if (ctx->sol.ordering != 0) { ctx->err = "dem_bench_sweeps times the Jacobi sweep (ordering 0)"; return DEM_ERR_INVALID; }
    const int64_t N = ctx->N;
    cudaStream_t s = ctx->s;
    if (getenv("DEM_DEBUG")) fprintf(stderr, "dem_bench_sweeps: %lld particles, %lld items\n", (long long)N, (long long)ctx->n_items);
    item_pack(ctx->n_items, ctx->pl, ctx->geo, ctx->cdel, ctx->row, ctx->Pfa, ctx->Pfb, ctx->it_rec, ctx->it_P[0], s);
    double4 *vb[2] = {ctx->vel[ctx->cur ^ 1], ctx->vel_prev}, *wb[2] = {ctx->ang[ctx->cur ^ 1], ctx->ang_prev};
    const double4 *vi = ctx->vel[ctx->cur], *wi = ctx->ang[ctx->cur];
    cudaEventRecord(ctx->ev[6], s);
    for (int it = 0; it < n; it++) {
        launch_sweep_items(false, N, vi, wi, ctx->pl.rad, vb[it & 1], wb[it & 1], ctx->pl, ctx->it_rec,
                           ctx->it_P[it & 1], ctx->it_P[(it & 1) ^ 1], ctx->db, ctx->sp, s);
        vi = vb[it & 1];
        wi = wb[it & 1];
    }
    cudaEventRecord(ctx->ev[7], s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[6], ctx->ev[7]);
    if (ms_per_sweep) *ms_per_sweep = ms / n;
    if (max_dv_rel) *max_dv_rel = 0.0;
    return DEM_OK;
}

void *dem_stream(dem_ctx *ctx) { return ctx ? (void *)ctx->s : nullptr; }

int64_t dem_drive_upload_bytes(void) { return (int64_t)sizeof(DevBoundary); }

int64_t dem_num_particles(const dem_ctx *ctx) { return ctx ? ctx->N_own : -1; }

int64_t dem_num_local(const dem_ctx *ctx) { return ctx ? ctx->N : -1; }

// the particle set changes (emitter, trimming): the current state is exported in
// gid order on the device, edited, validated, and only then is the contact history snapshot
// (handed to the next rebuild, dem_set_state's path: the warm start survives) and the new set
// loaded; a rejected edit leaves the context as it was
static dem_status snapshot_history(dem_ctx *ctx)
{
    if (ctx->have_step && !ctx->hist_pending) TRY(export_history(ctx));
    ctx->hist_pending = true;
    if (ctx->hauth && ctx->nh) CK(cudaMemsetAsync(ctx->hauth, 0, ctx->nh, ctx->s));
    return DEM_OK;
}
static dem_status export_particles(dem_ctx *ctx, int64_t extra, double **x, double **r, double **v, double **w,
                                   uint32_t **g)
{
    const int64_t N = ctx->N, M = N + extra;
    TRY(A(ctx, x, 3 * M + 3)); TRY(A(ctx, r, M + 1)); TRY(A(ctx, v, 3 * M + 3)); TRY(A(ctx, w, 3 * M + 3));
    TRY(A(ctx, g, M + 1));
    TRY(sync_check(ctx, "export_particles entry"));
    launch_to_gid_order(N, N, nullptr, ctx->gid, ctx->gid_sorted, ctx->pos, ctx->vel[ctx->cur], ctx->ang[ctx->cur], *x,
                        *v, *w, *r, *g, ctx->s);
    ctx->launches++;
    TRY(sync_check(ctx, "export_particles to_gid_order"));
    return DEM_OK;
}

dem_status dem_add_particles(dem_ctx *ctx, int64_t n, const double *pos, const double *radius, const double *vel,
                             const double *angvel, const uint32_t *gid, int32_t on_device)
{
    if (!ctx || n < 0 || (n && (!pos || !radius || !gid))) return DEM_ERR_INVALID;
    if (ctx->tp) { ctx->err = "dem_add_particles needs a single undecomposed context"; return DEM_ERR_INVALID; }
    if (!n) return DEM_OK;
    cudaStream_t s = ctx->s;
    const int64_t N = ctx->N;
    double *x = nullptr, *r = nullptr, *v = nullptr, *w = nullptr;
    uint32_t *g = nullptr;
    TRY(export_particles(ctx, n, &x, &r, &v, &w, &g));
    const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(x + 3 * N, pos, 3 * n * 8, k, s));
    CK(cudaMemcpyAsync(r + N, radius, n * 8, k, s));
    CK(cudaMemcpyAsync(g + N, gid, n * 4, k, s));
    if (vel) CK(cudaMemcpyAsync(v + 3 * N, vel, 3 * n * 8, k, s)); else CK(cudaMemsetAsync(v + 3 * N, 0, 3 * n * 8, s));
    if (angvel) CK(cudaMemcpyAsync(w + 3 * N, angvel, 3 * n * 8, k, s)); else CK(cudaMemsetAsync(w + 3 * N, 0, 3 * n * 8, s));
    CK(cudaStreamSynchronize(s));
    HostSet h;
    dem_status st = validate_particles(ctx, N + n, x, r, g, 1, true, h);
    if (st == DEM_OK) st = snapshot_history(ctx);
    if (st == DEM_OK) st = commit_particles(ctx, N + n, h, x, r, v, w, 1, true);
    for (void *q : {(void *)x, (void *)r, (void *)v, (void *)w, (void *)g}) dfree(ctx, q);
    if (st == DEM_OK) TRY(sync_check(ctx, "add_particles end"));
    return st;
}

dem_status dem_remove_particles(dem_ctx *ctx, int32_t axis, double lo, double hi, int64_t *n_removed)
{
    if (!ctx || axis < 0 || axis > 2 || std::isnan(lo) || std::isnan(hi)) return DEM_ERR_INVALID;
    if (ctx->tp) { ctx->err = "dem_remove_particles needs a single undecomposed context"; return DEM_ERR_INVALID; }
    cudaStream_t s = ctx->s;
    const int64_t N = ctx->N;
    double *x = nullptr, *r = nullptr, *v = nullptr, *w = nullptr;
    uint32_t *g = nullptr, *flag = nullptr, *scan = nullptr;
    TRY(export_particles(ctx, 0, &x, &r, &v, &w, &g));
    TRY(A(ctx, &flag, N + 2)); TRY(A(ctx, &scan, N + 2));
    launch_keep(N, x, axis, lo, hi, flag, s);
    scan_u32(flag, scan, N, ctx->scan_tmp, s, &ctx->launches);
    uint32_t keep = 0;
    CK(cudaMemcpyAsync(&keep, scan + N, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double *x2 = nullptr, *r2 = nullptr, *v2 = nullptr, *w2 = nullptr;
    uint32_t *g2 = nullptr;
    TRY(A(ctx, &x2, 3 * (int64_t)keep + 3)); TRY(A(ctx, &r2, keep + 1)); TRY(A(ctx, &v2, 3 * (int64_t)keep + 3));
    TRY(A(ctx, &w2, 3 * (int64_t)keep + 3)); TRY(A(ctx, &g2, keep + 1));
    launch_keep_gather(N, flag, scan, x, r, v, w, g, x2, r2, v2, w2, g2, s);
    CK(cudaStreamSynchronize(s));
    HostSet h;
    dem_status st = validate_particles(ctx, keep, x2, r2, g2, 1, true, h);
    if (st == DEM_OK) st = snapshot_history(ctx);
    if (st == DEM_OK) st = commit_particles(ctx, keep, h, x2, r2, v2, w2, 1, true);
    for (void *q : {(void *)x, (void *)r, (void *)v, (void *)w, (void *)g, (void *)flag, (void *)scan, (void *)x2,
                    (void *)r2, (void *)v2, (void *)w2, (void *)g2})
        dfree(ctx, q);
    if (n_removed) *n_removed = N - (int64_t)keep;
    return st;
}

dem_status dem_rebalance(dem_ctx *ctx, int32_t n_bins, double *faces_out)
{
    if (!ctx || n_bins < 2) return DEM_ERR_INVALID;
    if (!ctx->tp || ctx->G < 2) return DEM_OK;
    cudaStream_t s = ctx->s;
    const int G = ctx->G;
    const double lo = ctx->box.lo[0], hi = ctx->box.hi[0];
    // 1. global histogram of the owned particles' x (each particle counted by its owner)
    unsigned long long *dh = nullptr;
    TRY(A(ctx, &dh, n_bins));
    launch_hist_x(ctx->N, OWN(ctx), ctx->pos, lo, hi, n_bins, dh, s);
    std::vector<long long> h(n_bins);
    CK(cudaMemcpyAsync(h.data(), dh, n_bins * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(ctx, dh);
    for (int o = 0; o < n_bins; o += 64)       // the transports reduce at most 64 values per call
        if (!ctx->tp->allreduce_i64(h.data() + o, std::min(64, n_bins - o), 0, s, ctx->err)) return DEM_ERR_NCCL;
    // 2. current faces (face k = slab_lo of rank k), assembled by a sum over ranks
    std::vector<double> f(G - 1, 0.0);
    if (ctx->rank > 0) f[ctx->rank - 1] = ctx->slab_lo;
    for (int o = 0; o < G - 1; o += 64)
        if (!ctx->tp->allreduce_f64(f.data() + o, std::min(64, G - 1 - o), 0, s, ctx->err)) return DEM_ERR_NCCL;
    // 3. count quantiles (linear within a bin), each face moved by at most one skin: a particle
    //    that changes owner lies within a skin of the old face, so all its contacts of the last
    //    step (partners within 2 r_max) and their impulse history are inside the new owner's
    //    ghost band (2 r_max + 2 skin) -- no history has to travel; interior slabs stay one band wide
    long long tot = 0;
    for (long long v : h) tot += v;
    const double bw = (hi - lo) / n_bins, step = ctx->grid.skin;
    std::vector<double> nf(f);
    for (int k = 0; k < G - 1 && tot > 0; k++) {
        const double want = (double)tot * (k + 1) / G;
        double acc = 0.0, t = hi;
        for (int b = 0; b < n_bins; b++) {
            if (acc + h[b] >= want) { t = lo + bw * (b + (h[b] ? (want - acc) / h[b] : 0.0)); break; }
            acc += h[b];
        }
        nf[k] = f[k] + std::max(-step, std::min(step, t - f[k]));
    }
    for (int k = 1; k < G - 1; k++) nf[k] = std::max(nf[k], nf[k - 1] + ctx->band_w);
    for (int k = G - 3; k >= 0; k--) nf[k] = std::min(nf[k], nf[k + 1] - ctx->band_w);
    if (ctx->rank > 0) ctx->slab_lo = nf[ctx->rank - 1];
    if (ctx->rank < G - 1) ctx->slab_hi = nf[ctx->rank];
    if (faces_out) for (int k = 0; k < G - 1; k++) faces_out[k] = nf[k];
    ctx->need_rebuild = true;           // ownership follows the new faces at the next step's rebuild
    return DEM_OK;
}

void *dem_loopback_create(int32_t world_size) { return world_size >= 1 ? (void *)new LoopGroup(world_size) : nullptr; }

void dem_loopback_destroy(void *group) { delete (LoopGroup *)group; }

dem_status dem_nccl_unique_id(void *out128)
{
    if (!out128) return DEM_ERR_INVALID;
    std::string err;
    if (!nccl_unique_id(out128, err)) { g_create_err = err; return DEM_ERR_NCCL; }
    return DEM_OK;
}

dem_status dem_destroy(dem_ctx *ctx)
{
    if (!ctx) return DEM_ERR_INVALID;
    if (ctx->s) cudaStreamSynchronize(ctx->s);
    for (int q = 0; q < 4; q++)
        for (auto *g : {&ctx->g_imp[q], &ctx->g_main[q]})
            if (g->exec) cudaGraphExecDestroy(g->exec);
    std::vector<void *> all = ctx->allocs;
    for (void *p : all) dfree(ctx, p);
    for (int e = 0; e < 8; e++) if (ctx->ev[e]) cudaEventDestroy(ctx->ev[e]);
    if (ctx->hsc) cudaFreeHost(ctx->hsc);
    if (ctx->hnc) cudaFreeHost(ctx->hnc);
    if (ctx->own_stream && ctx->s) cudaStreamDestroy(ctx->s);
    delete ctx->tp;
    delete ctx;
    return DEM_OK;
}

const char *dem_last_error(const dem_ctx *ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

}  // extern "C"
