// detect.cu -- contact detection for the DEM step ("re-computed at every simulation
// timestep using a collision detection algorithm"), north_star subsystems (a)-(c):
//
//  rebuild (when the Verlet skin is used up):
//    k_keys        level (factor-2 size class) + Morton key of the particle's cell in its level
//    radix sort    (radix_sort.cu) and k_permute of the SoA particle state (32 B vector loads)
//    k_cells       dense per-level cell tables [start, end) over the sorted order
//    k_broad       multi-level grid search: own level 27 cells, coarser levels only from the
//                  finer side (a fine particle never scans a coarse-cell neighbourhood of fine
//                  particles, and coarse particles never scan fine grids); walls, plate boxes
//    k_trans_*     transposed candidate lists (incoming half-contacts) in deterministic order
//    k_hist_*      sorted-key merge that carries the impulse history (P_n, P_t, P_r) across a
//                  rebuild by binary search of the (gid_a, gid_b) key
//  every step:
//    k_narrow      exact fp64 contact predicate with a fixed IEEE operation sequence
//    k_compact     compaction of active candidates into the contact arrays + warm start
//    k_inc_*       half-contact CSR per particle (deterministic order)
#include "common.cuh"
#include "kernels.h"

// ------------------------------------------------------------------ exact contact geometry
// Returns 1 contact, 0 none, -1 degenerate (coincident centres, flagged and skipped).
// The predicate is exact fp64 with a fixed operation order (reading R14); n and delta of an
// active pair come from pair_geom, the sequence the sweeps re-evaluate (common.cuh).
__device__ __forceinline__ int contact_geom(uint2 ij, const double4 *__restrict__ pos, const DevBoundary *bnd,
                                            d3 &n, double &delta)
{
    const double4 A = pos[ij.x];
    if (!(ij.y & PARTNER_EXT)) {
        const double4 B = pos[ij.y];
        const double dx = __dsub_rn(B.x, A.x), dy = __dsub_rn(B.y, A.y), dz = __dsub_rn(B.z, A.z);
        const double d2 = dist2_rn(dx, dy, dz);
        const double R = __dadd_rn(A.w, B.w);
        if (!(d2 < __dmul_rn(R, R))) return 0;
        if (d2 == 0.0) return -1;
        pair_geom(A, B, n, delta);
        return 1;
    }
    return ext_geom(A, ij.y & ~PARTNER_EXT, bnd, n, delta);
}

// ------------------------------------------------------------------ rebuild kernels
__global__ void k_keys(int64_t N, const double4 *__restrict__ pos, GridParams g, uint64_t *__restrict__ keys,
                       uint32_t *__restrict__ vals)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double4 p = pos[i];
    const int L = level_of(p.w, g.rmin, g.nlev);
    const GridLevel &lv = g.lv[L];
    const int cx = cell_coord(p.x, lv.ox, lv.cell, lv.nx);
    const int cy = cell_coord(p.y, lv.oy, lv.cell, lv.ny);
    const int cz = cell_coord(p.z, lv.oz, lv.cell, lv.nz);
    const uint64_t m = spread3((uint32_t)cx) | (spread3((uint32_t)cy) << 1) | (spread3((uint32_t)cz) << 2);
    keys[i] = ((uint64_t)L << (3 * g.bits)) | m;
    vals[i] = (uint32_t)i;
}

__global__ void k_permute(int64_t N, const uint32_t *__restrict__ idx, const double4 *__restrict__ pin,
                          const double4 *__restrict__ vin, const double4 *__restrict__ win,
                          const uint32_t *__restrict__ gin, double4 *__restrict__ pout, double4 *__restrict__ vout,
                          double4 *__restrict__ wout, uint32_t *__restrict__ gout)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t s = idx[i];
    pout[i] = pin[s];
    vout[i] = vin[s];
    wout[i] = win[s];
    gout[i] = gin[s];
}

__device__ __forceinline__ uint64_t cell_slot(const GridParams &g, uint64_t key)
{
    const int L = (int)(key >> (3 * g.bits));
    const uint64_t m = key & ((1ULL << (3 * g.bits)) - 1);
    const uint32_t cx = compact3(m), cy = compact3(m >> 1), cz = compact3(m >> 2);
    const GridLevel &lv = g.lv[L];
    return lv.offset + (uint64_t)cx + (uint64_t)lv.nx * ((uint64_t)cy + (uint64_t)lv.ny * (uint64_t)cz);
}

__global__ void k_cells(int64_t N, const uint64_t *__restrict__ keys, GridParams g, uint32_t *__restrict__ cstart,
                        uint32_t *__restrict__ cend)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint64_t k = keys[i];
    const uint64_t slot = cell_slot(g, k);
    if (i == 0 || keys[i - 1] != k) cstart[slot] = (uint32_t)i;
    if (i == N - 1 || keys[i + 1] != k) cend[slot] = (uint32_t)(i + 1);
}

// Multi-level broad phase.  FILL = false counts candidates per particle, FILL = true writes
// them at co_start[i] in the same deterministic order.
template <bool FILL>
__global__ void k_broad(int64_t N, const double4 *__restrict__ pos, GridParams g, const uint32_t *__restrict__ cstart,
                        const uint32_t *__restrict__ cend, const DevBoundary *__restrict__ bnd,
                        uint32_t *__restrict__ cnt_or_start, uint2 *__restrict__ cand)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double4 p = pos[i];
    const double skin = g.skin;
    const int L = level_of(p.w, g.rmin, g.nlev);
    uint32_t c = 0;
    uint32_t base = FILL ? cnt_or_start[i] : 0u;
    auto emit = [&](uint32_t j) {
        if (FILL) cand[base + c] = make_uint2((uint32_t)i, j);
        c++;
    };
    for (int Lq = L; Lq < g.nlev; Lq++) {
        const GridLevel &lv = g.lv[Lq];
        if (!lv.present) continue;
        // search box: own level -> the 27 neighbour cells; coarser level -> the cells that
        // overlap the AABB inflated by r_max(L') + skin (<= 3 per axis since cell >= extent)
        const double ext = (Lq == L) ? lv.cell : (p.w + lv.rmax + skin);
        int lo[3], hi[3];
        const double pc[3] = {p.x, p.y, p.z}, oc[3] = {lv.ox, lv.oy, lv.oz};
        const int nc[3] = {lv.nx, lv.ny, lv.nz};
        for (int k = 0; k < 3; k++) {
            if (Lq == L) {
                const int cc = cell_coord(pc[k], oc[k], lv.cell, nc[k]);
                lo[k] = max(cc - 1, 0);
                hi[k] = min(cc + 1, nc[k] - 1);
            } else {
                lo[k] = cell_coord(pc[k] - ext, oc[k], lv.cell, nc[k]);
                hi[k] = cell_coord(pc[k] + ext, oc[k], lv.cell, nc[k]);
            }
        }
        for (int cz = lo[2]; cz <= hi[2]; cz++)
            for (int cy = lo[1]; cy <= hi[1]; cy++)
                for (int cx = lo[0]; cx <= hi[0]; cx++) {
                    const uint64_t slot = lv.offset + (uint64_t)cx + (uint64_t)lv.nx * ((uint64_t)cy + (uint64_t)lv.ny * (uint64_t)cz);
                    const uint32_t s = cstart[slot], e = cend[slot];
                    for (uint32_t j = s; j < e; j++) {
                        if (j <= (uint32_t)i) continue;
                        const double4 q = pos[j];
                        const double dx = q.x - p.x, dy = q.y - p.y, dz = q.z - p.z;
                        const double R = p.w + q.w + skin;
                        if (dx * dx + dy * dy + dz * dz < R * R) emit(j);
                    }
                }
    }
    // box walls: signed distance < r + skin
    for (int w = 0; w < 6; w++) {
        if (!bnd->wpresent[w]) continue;
        const double s = (p.x - bnd->wp[w][0]) * bnd->wn[w][0] + (p.y - bnd->wp[w][1]) * bnd->wn[w][1] +
                         (p.z - bnd->wp[w][2]) * bnd->wn[w][2];
        if (s < p.w + skin) emit(PARTNER_EXT | (uint32_t)w);
    }
    // plate boxes: distance to the box < r + skin
    for (int q = 0; q < bnd->n_plates; q++)
        for (int b = 0; b < bnd->nbox[q]; b++) {
            double d2 = 0.0;
            const double pc[3] = {p.x, p.y, p.z};
            for (int k = 0; k < 3; k++) {
                const double lo = bnd->ppos[q][k] + bnd->lo[q][b][k], hi = bnd->ppos[q][k] + bnd->hi[q][b][k];
                const double dd = pc[k] < lo ? lo - pc[k] : (pc[k] > hi ? pc[k] - hi : 0.0);
                d2 += dd * dd;
            }
            const double R = p.w + skin;
            if (d2 < R * R) emit(PARTNER_EXT | PARTNER_PLATE | ((uint32_t)q << 4) | (uint32_t)b);
        }
    if (!FILL) cnt_or_start[i] = c;
}

__global__ void k_trans_count(int64_t nc, const uint2 *__restrict__ cand, uint32_t *__restrict__ cnt)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nc) return;
    const uint32_t j = cand[k].y;
    if (!(j & PARTNER_EXT)) atomicAdd(&cnt[j], 1u);
}

__global__ void k_trans_fill(int64_t nc, const uint2 *__restrict__ cand, const uint32_t *__restrict__ ct_start,
                             uint32_t *__restrict__ cursor, uint32_t *__restrict__ ct_list)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nc) return;
    const uint32_t j = cand[k].y;
    if (!(j & PARTNER_EXT)) ct_list[ct_start[j] + atomicAdd(&cursor[j], 1u)] = (uint32_t)k;
}

// sort each particle's incoming list by candidate index (= by partner, since candidates are
// ordered by owner): makes the order independent of the atomic fill order
__global__ void k_trans_sort(int64_t N, const uint32_t *__restrict__ ct_start, uint32_t *__restrict__ ct_list)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t s = ct_start[i], e = ct_start[i + 1];
    for (uint32_t a = s + 1; a < e; a++) {
        const uint32_t v = ct_list[a];
        uint32_t b = a;
        while (b > s && ct_list[b - 1] > v) { ct_list[b] = ct_list[b - 1]; b--; }
        ct_list[b] = v;
    }
}

// public key of a candidate and whether the GPU orientation (i, j) is flipped w.r.t. the
// canonical one (a = smaller gid)
__device__ __forceinline__ uint64_t cand_key(uint2 ij, const uint32_t *__restrict__ gid, bool &flip)
{
    const uint32_t gi = gid[ij.x];
    flip = false;
    if (ij.y & PARTNER_EXT) {
        const uint32_t code = ij.y & ~PARTNER_EXT;
        uint32_t kb = (code & PARTNER_PLATE) ? PLATE_KEY_BASE + 16u * ((code >> 4) & 0xF) + (code & 0xF)
                                             : WALL_KEY_BASE + code;
        return ((uint64_t)gi << 32) | kb;
    }
    const uint32_t gj = gid[ij.y];
    if (gj < gi) { flip = true; return ((uint64_t)gj << 32) | gi; }
    return ((uint64_t)gi << 32) | gj;
}

__global__ void k_hist_flag(int64_t nc, const P4 *__restrict__ Pa, const P4 *__restrict__ Pb,
                            uint32_t *__restrict__ flag)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nc) return;
    const P4 a = Pa[k], b = Pb[k];
    flag[k] = (a.x != 0 || a.y != 0 || a.z != 0 || a.w != 0 || b.x != 0 || b.y != 0 || b.z != 0) ? 1u : 0u;
}

__global__ void k_hist_keys(int64_t nc, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ scan,
                            const uint2 *__restrict__ cand, const uint32_t *__restrict__ gid, uint64_t *__restrict__ keys,
                            uint32_t *__restrict__ vals)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nc || !flag[k]) return;
    bool flip;
    keys[scan[k]] = cand_key(cand[k], gid, flip);
    vals[scan[k]] = (uint32_t)k;
}

// gather P of the sorted history into canonical orientation
__global__ void k_hist_gather(int64_t nh, const uint32_t *__restrict__ vals, const uint2 *__restrict__ cand,
                              const uint32_t *__restrict__ gid, const P4 *__restrict__ Pa,
                              const P4 *__restrict__ Pb, P4 *__restrict__ hPa, P4 *__restrict__ hPb)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nh) return;
    const uint32_t k = vals[t];
    bool flip;
    cand_key(cand[k], gid, flip);
    P4 a = Pa[k], b = Pb[k];
    if (flip) { a.y = -a.y; a.z = -a.z; a.w = -a.w; b.x = -b.x; b.y = -b.y; b.z = -b.z; }
    hPa[t] = a;
    hPb[t] = b;
}

// new candidates pick up history by binary search of their key in the sorted history
__global__ void k_hist_carry(int64_t nc, const uint2 *__restrict__ cand, const uint32_t *__restrict__ gid,
                             const uint64_t *__restrict__ hkey, const P4 *__restrict__ hPa,
                             const P4 *__restrict__ hPb, int64_t nh, P4 *__restrict__ Pa,
                             P4 *__restrict__ Pb)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nc) return;
    bool flip;
    const uint64_t key = cand_key(cand[k], gid, flip);
    int64_t lo = 0, hi = nh;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (hkey[mid] < key) lo = mid + 1; else hi = mid;
    }
    P4 a = mkP4(0, 0, 0, 0), b = a;
    if (lo < nh && hkey[lo] == key) {
        a = hPa[lo];
        b = hPb[lo];
        if (flip) { a.y = -a.y; a.z = -a.z; a.w = -a.w; b.x = -b.x; b.y = -b.y; b.z = -b.z; }
    }
    Pa[k] = a;
    Pb[k] = b;
}

// ------------------------------------------------------------------ per-step kernels
__global__ void k_narrow(int64_t nc, const uint2 *__restrict__ cand, const double4 *__restrict__ pos,
                         const DevBoundary *__restrict__ bnd, uint32_t *__restrict__ flag, P4 *__restrict__ Pa,
                         P4 *__restrict__ Pb, StepScalars *sc)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nc) return;
    d3 n;
    double delta;
    const int r = contact_geom(cand[k], pos, bnd, n, delta);
    flag[k] = r == 1 ? 1u : 0u;
    if (r != 1) {
        Pa[k] = mkP4(0, 0, 0, 0);
        Pb[k] = mkP4(0, 0, 0, 0);
    }
    if (r == -1) atomicAdd(&sc->n_degenerate, 1u);
}

__device__ __forceinline__ void partner_mu(uint32_t j, const SolveParams &sp, const DevBoundary *bnd, double &mt,
                                           double &mr)
{
    if (!(j & PARTNER_EXT)) { mt = sp.mu_t; mr = sp.mu_r; return; }
    const uint32_t code = j & ~PARTNER_EXT;
    if (code & PARTNER_PLATE) { const int p = (code >> 4) & 0xF; mt = bnd->pmu_t[p]; mr = bnd->pmu_r[p]; }
    else { mt = bnd->wall_mu_t; mr = bnd->wall_mu_r; }
}

__global__ void k_compact(int64_t nc, const uint2 *__restrict__ cand, const uint32_t *__restrict__ flag,
                          const uint32_t *__restrict__ scan, const double4 *__restrict__ pos,
                          const DevBoundary *__restrict__ bnd, SolveParams sp, const P4 *__restrict__ Pca,
                          const P4 *__restrict__ Pcb, uint2 *__restrict__ cij, G4 *__restrict__ geo,
                          R4 *__restrict__ row, double *__restrict__ cdel, P4 *__restrict__ Pa, P4 *__restrict__ Pb,
                          uint32_t *__restrict__ ccand, const uint32_t *__restrict__ gid, StepScalars *sc)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nc || !flag[k]) return;
    const uint32_t c = scan[k];
    // canonical orientation: a = smaller gid (the candidate may hold the pair either way)
    const bool flip = cand_flip(cand[k], gid);
    const uint2 ij = flip ? make_uint2(cand[k].y, cand[k].x) : cand[k];
    d3 n;
    double delta;
    contact_geom(ij, pos, bnd, n, delta);
    const double ra = pos[ij.x].w;
    const bool ext = (ij.y & PARTNER_EXT) != 0;
    const double rb = ext ? 0.0 : pos[ij.y].w;
    const double Rs = ext ? ra : rstar(ra, rb);
    cij[c] = ij;
    double mt, mr;
    partner_mu(ij.y, sp, bnd, mt, mr);
    const G4 gf = mkG4(n.x, n.y, n.z, mr * Rs);
    geo[c] = gf;
    row[c] = mkR4(0, 0, ra - 0.5 * delta, ext ? 0.0 : rb - 0.5 * delta);
    cdel[c] = delta;
    ccand[c] = (uint32_t)k | (flip ? CCAND_FLIP : 0u);
    // warm start (reading R12): re-project P_t onto the new tangent plane, clamp cones
    // (candidate-slot impulses are kept in candidate orientation: flip to canonical)
    P4 A = Pca[k], B = Pcb[k];
    if (flip) { A.y = -A.y; A.z = -A.z; A.w = -A.w; B.x = -B.x; B.y = -B.y; B.z = -B.z; }
    const d3 nf = mk(gf.x, gf.y, gf.z);
    double Pn = A.x > 0 ? (double)A.x : 0.0;
    d3 Pt = mk(A.y, A.z, A.w), Pr = mk(B.x, B.y, B.z);
    Pt = Pt - dot(Pt, nf) * nf;
    if (sp.rolling_dims == 2) Pr = Pr - dot(Pr, nf) * nf;
    double lim = mt * Pn, m2 = dot(Pt, Pt);
    if (m2 > lim * lim) { const double s = m2 > 0.0 ? lim / sqrt(m2) : 0.0; Pt = s * Pt; }
    lim = mr * Rs * Pn;
    m2 = dot(Pr, Pr);
    if (m2 > lim * lim) { const double s = m2 > 0.0 ? lim / sqrt(m2) : 0.0; Pr = s * Pr; }
    Pa[c] = mkP4(Pn, Pt.x, Pt.y, Pt.z);
    Pb[c] = mkP4(Pr.x, Pr.y, Pr.z, 0);
}

// per-kind contact counts: grid-stride warp ballots, block sums in shared memory, one atomic per
// block and kind (one atomic per warp serialised 1.4 M updates on one address: ~1 ms)
// A contact is counted by the rank that owns its particle with the smaller gid (boundary
// contacts: the rank owning the particle), so sums over ranks count each contact once.
__global__ void __launch_bounds__(256) k_count_kinds(int64_t nc, const uint8_t *__restrict__ own,
                                                     const uint2 *__restrict__ cij, const uint32_t *__restrict__ gid,
                                                     StepScalars *sc)
{
    __shared__ unsigned sm[3][8];
    unsigned npp = 0, npl = 0, nwl = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x; c0 < nc; c0 += stride) {   // warp-uniform trip count
        const int64_t c = c0 + threadIdx.x;
        const uint2 ij = c < nc ? cij[c] : make_uint2(0, 0);
        const uint32_t j = ij.y;
        bool ok = c < nc;
        if (ok) {
            const uint32_t o = (j & PARTNER_EXT) ? ij.x : (gid[ij.x] < gid[j] ? ij.x : j);
            ok = !own || own[o];
        }
        npp += __popc(__ballot_sync(0xffffffffu, ok && !(j & PARTNER_EXT)));
        npl += __popc(__ballot_sync(0xffffffffu, ok && (j & PARTNER_EXT) && (j & PARTNER_PLATE)));
        nwl += __popc(__ballot_sync(0xffffffffu, ok && (j & PARTNER_EXT) && !(j & PARTNER_PLATE)));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sm[0][w] = npp; sm[1][w] = npl; sm[2][w] = nwl; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); q++) { npp += sm[0][q]; npl += sm[1][q]; nwl += sm[2][q]; }
        if (npp) atomicAdd(&sc->n_pp, npp);
        if (npl) atomicAdd(&sc->n_plate, npl);
        if (nwl) atomicAdd(&sc->n_wall, nwl);
    }
}

__global__ void k_inc_count(int64_t N, const uint32_t *__restrict__ co_start, const uint32_t *__restrict__ scan,
                            const uint32_t *__restrict__ ct_start, const uint32_t *__restrict__ ct_list,
                            const uint32_t *__restrict__ flag, uint32_t *__restrict__ cnt)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    uint32_t c = scan[co_start[i + 1]] - scan[co_start[i]];
    for (uint32_t t = ct_start[i]; t < ct_start[i + 1]; t++) c += flag[ct_list[t]];
    cnt[i] = c;
}

// A particle's half-contacts in the order of their partners' gids (boundary bodies last): the
// per-particle reduction order is then the same in every decomposition.
__global__ void k_inc_fill(int64_t N, const uint32_t *__restrict__ co_start, const uint2 *__restrict__ cand,
                           const uint32_t *__restrict__ scan, const uint32_t *__restrict__ ct_start,
                           const uint32_t *__restrict__ ct_list, const uint32_t *__restrict__ flag,
                           const uint32_t *__restrict__ gid, const uint32_t *__restrict__ inc_start,
                           uint2 *__restrict__ inc)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const uint32_t s = inc_start[i];
    uint32_t o = s;
    for (uint32_t t = ct_start[i]; t < ct_start[i + 1]; t++) {       // i is the candidate's j
        const uint32_t k = ct_list[t];
        if (flag[k]) inc[o++] = make_uint2(scan[k] | (cand_flip(cand[k], gid) ? 0u : B_SIDE), cand[k].x);
    }
    for (uint32_t k = co_start[i]; k < co_start[i + 1]; k++)        // i is the candidate's i
        if (flag[k]) inc[o++] = make_uint2(scan[k] | (cand_flip(cand[k], gid) ? B_SIDE : 0u), cand[k].y);
    for (uint32_t a = s + 1; a < o; a++) {                           // insertion sort by partner
        const uint2 v = inc[a];
        const uint64_t kv = partner_key(v.y, gid);
        uint32_t b = a;
        while (b > s && partner_key(inc[b - 1].y, gid) > kv) { inc[b] = inc[b - 1]; b--; }
        inc[b] = v;
    }
}

// divergence diagnostics: the smallest public key among contacts with a non-finite
// impulse, else the smallest gid among particles with a non-finite state (key = gid << 32 | ~0)
__global__ void k_first_bad(int64_t nc, int64_t N, const uint8_t *__restrict__ own, const uint2 *__restrict__ cij,
                            const uint32_t *__restrict__ gid, const P4 *__restrict__ Pa, const P4 *__restrict__ Pb,
                            const double4 *__restrict__ pos, const double4 *__restrict__ vel,
                            const double4 *__restrict__ ang, unsigned long long *out)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nc) {
        const P4 a = Pa[t], b = Pb[t];
        const bool bad = !isfinite(a.x) || !isfinite(a.y) || !isfinite(a.z) || !isfinite(a.w) || !isfinite(b.x) ||
                         !isfinite(b.y) || !isfinite(b.z);
        if (bad && (!own || own[cij[t].x])) {
            bool flip;
            atomicMin(&out[0], (unsigned long long)cand_key(cij[t], gid, flip));
        }
    }
    if (t < N && (!own || own[t])) {
        const double4 x = pos[t], v = vel[t], w = ang[t];
        if (!isfinite(x.x + x.y + x.z) || !isfinite(v.x + v.y + v.z) || !isfinite(w.x + w.y + w.z))
            atomicMin(&out[1], ((unsigned long long)gid[t] << 32) | 0xFFFFFFFFull);
    }
}
void launch_first_bad(int64_t nc, int64_t N, const uint8_t *own, const uint2 *cij, const uint32_t *gid, const P4 *Pa,
                      const P4 *Pb, const double4 *pos, const double4 *vel, const double4 *ang,
                      unsigned long long *out, cudaStream_t s)
{
    cudaMemsetAsync(out, 0xFF, 2 * sizeof(unsigned long long), s);
    const int64_t n = nc > N ? nc : N;
    if (n) k_first_bad<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nc, N, own, cij, gid, Pa, Pb, pos, vel, ang, out);
}

// ------------------------------------------------------------------ output helpers
// contacts -> public keys (canonical orientation), values = contact index
// contacts reported by this rank (owner of the smaller gid; boundary contacts: the particle's
// owner) get their public key, the others sort last (key ~0); cnt counts the reported ones
__global__ void k_contact_keys(int64_t nc, const uint8_t *__restrict__ own, const uint2 *__restrict__ cij,
                               const uint32_t *__restrict__ gid, uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
                               unsigned int *cnt)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    bool flip;
    const uint2 ij = cij[c];
    const uint32_t o = (ij.y & PARTNER_EXT) ? ij.x : (gid[ij.x] < gid[ij.y] ? ij.x : ij.y);
    const bool mine = !own || own[o];
    keys[c] = mine ? cand_key(ij, gid, flip) : ~0ull;
    vals[c] = (uint32_t)c;
    if (mine) atomicAdd(cnt, 1u);
}

__global__ void k_contact_out(int64_t nc, const uint32_t *__restrict__ vals, const uint2 *__restrict__ cij,
                              const uint32_t *__restrict__ gid, const G4 *__restrict__ geo, const double *__restrict__ cdel,
                              const P4 *__restrict__ Pa, const P4 *__restrict__ Pb, double *__restrict__ nrm,
                              double *__restrict__ delta, double *__restrict__ P)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nc) return;
    const uint32_t c = vals[t];
    bool flip;
    cand_key(cij[c], gid, flip);
    const double s = flip ? -1.0 : 1.0;
    const G4 g = geo[c];
    const P4 a = Pa[c], b = Pb[c];
    if (nrm) { nrm[3 * t] = s * g.x; nrm[3 * t + 1] = s * g.y; nrm[3 * t + 2] = s * g.z; }
    if (delta) delta[t] = cdel[c];
    if (P) {
        P[7 * t] = a.x;
        P[7 * t + 1] = s * a.y; P[7 * t + 2] = s * a.z; P[7 * t + 3] = s * a.w;
        P[7 * t + 4] = s * b.x; P[7 * t + 5] = s * b.y; P[7 * t + 6] = s * b.z;
    }
}

// ------------------------------------------------------------------ launchers
#define GRID(n) (unsigned)(((n) + 255) / 256), 256, 0, s

void launch_keys(int64_t N, const double4 *pos, const GridParams &g, uint64_t *keys, uint32_t *vals, cudaStream_t s)
{ k_keys<<<GRID(N)>>>(N, pos, g, keys, vals); }
void launch_permute(int64_t N, const uint32_t *idx, const double4 *pin, const double4 *vin, const double4 *win,
                    const uint32_t *gin, double4 *pout, double4 *vout, double4 *wout, uint32_t *gout, cudaStream_t s)
{ k_permute<<<GRID(N)>>>(N, idx, pin, vin, win, gin, pout, vout, wout, gout); }
void launch_cells(int64_t N, const uint64_t *keys, const GridParams &g, uint32_t *cs, uint32_t *ce, cudaStream_t s)
{ k_cells<<<GRID(N)>>>(N, keys, g, cs, ce); }
void launch_broad(bool fill, int64_t N, const double4 *pos, const GridParams &g, const uint32_t *cs,
                  const uint32_t *ce, const DevBoundary *bnd, uint32_t *cnt_or_start, uint2 *cand, cudaStream_t s)
{
    if (fill) k_broad<true><<<GRID(N)>>>(N, pos, g, cs, ce, bnd, cnt_or_start, cand);
    else k_broad<false><<<GRID(N)>>>(N, pos, g, cs, ce, bnd, cnt_or_start, cand);
}
void launch_trans(int64_t N, int64_t nc, const uint2 *cand, uint32_t *cnt, uint32_t *ct_start, uint32_t *cursor,
                  uint32_t *ct_list, void *scan_tmp, cudaStream_t s, long long *launches)
{
    cudaMemsetAsync(cnt, 0, (N + 1) * sizeof(uint32_t), s);
    cudaMemsetAsync(cursor, 0, (N + 1) * sizeof(uint32_t), s);
    if (nc) k_trans_count<<<GRID(nc)>>>(nc, cand, cnt);
    scan_u32(cnt, ct_start, N, scan_tmp, s, launches);
    if (nc) k_trans_fill<<<GRID(nc)>>>(nc, cand, ct_start, cursor, ct_list);
    if (N) k_trans_sort<<<GRID(N)>>>(N, ct_start, ct_list);
    *launches += 3;
}
void launch_hist_flag(int64_t nc, const P4 *Pa, const P4 *Pb, uint32_t *flag, cudaStream_t s)
{ if (nc) k_hist_flag<<<GRID(nc)>>>(nc, Pa, Pb, flag); }
void launch_hist_keys(int64_t nc, const uint32_t *flag, const uint32_t *scan, const uint2 *cand, const uint32_t *gid,
                      uint64_t *keys, uint32_t *vals, cudaStream_t s)
{ if (nc) k_hist_keys<<<GRID(nc)>>>(nc, flag, scan, cand, gid, keys, vals); }
void launch_hist_gather(int64_t nh, const uint32_t *vals, const uint2 *cand, const uint32_t *gid, const P4 *Pa,
                        const P4 *Pb, P4 *hPa, P4 *hPb, cudaStream_t s)
{ if (nh) k_hist_gather<<<GRID(nh)>>>(nh, vals, cand, gid, Pa, Pb, hPa, hPb); }
void launch_hist_carry(int64_t nc, const uint2 *cand, const uint32_t *gid, const uint64_t *hkey, const P4 *hPa,
                       const P4 *hPb, int64_t nh, P4 *Pa, P4 *Pb, cudaStream_t s)
{ if (nc) k_hist_carry<<<GRID(nc)>>>(nc, cand, gid, hkey, hPa, hPb, nh, Pa, Pb); }
void launch_narrow(int64_t nc, const uint2 *cand, const double4 *pos, const DevBoundary *bnd, uint32_t *flag,
                   P4 *Pa, P4 *Pb, StepScalars *sc, cudaStream_t s)
{ if (nc) k_narrow<<<GRID(nc)>>>(nc, cand, pos, bnd, flag, Pa, Pb, sc); }
void launch_compact(int64_t nc, const uint2 *cand, const uint32_t *flag, const uint32_t *scan, const double4 *pos,
                    const DevBoundary *bnd, const SolveParams &sp, const P4 *Pca, const P4 *Pcb, uint2 *cij,
                    G4 *geo, R4 *row, double *cdel, P4 *Pa, P4 *Pb, uint32_t *ccand, const uint32_t *gid, StepScalars *sc,
                    cudaStream_t s)
{ if (nc) k_compact<<<GRID(nc)>>>(nc, cand, flag, scan, pos, bnd, sp, Pca, Pcb, cij, geo, row, cdel, Pa, Pb, ccand, gid, sc); }
void launch_count_kinds(int64_t nc, const uint8_t *own, const uint2 *cij, const uint32_t *gid, StepScalars *sc, cudaStream_t s)
{ if (nc) k_count_kinds<<<(unsigned)std::min<int64_t>((nc + 255) / 256, 148 * 8), 256, 0, s>>>(nc, own, cij, gid, sc); }
void launch_inc(int64_t N, const uint32_t *co_start, const uint2 *cand, const uint32_t *scan, const uint32_t *ct_start,
                const uint32_t *ct_list, const uint32_t *flag, const uint32_t *gid, uint32_t *cnt, uint32_t *inc_start,
                uint2 *inc, void *scan_tmp, cudaStream_t s, long long *launches)
{
    if (N) k_inc_count<<<GRID(N)>>>(N, co_start, scan, ct_start, ct_list, flag, cnt);
    scan_u32(cnt, inc_start, N, scan_tmp, s, launches);
    if (N) k_inc_fill<<<GRID(N)>>>(N, co_start, cand, scan, ct_start, ct_list, flag, gid, inc_start, inc);
    *launches += 2;
}
void launch_contact_keys(int64_t nc, const uint8_t *own, const uint2 *cij, const uint32_t *gid, uint64_t *keys, uint32_t *vals,
                         unsigned int *cnt, cudaStream_t s)
{ if (nc) k_contact_keys<<<GRID(nc)>>>(nc, own, cij, gid, keys, vals, cnt); }
void launch_contact_out(int64_t nc, const uint32_t *vals, const uint2 *cij, const uint32_t *gid, const G4 *geo,
                        const double *cdel, const P4 *Pa, const P4 *Pb, double *nrm, double *delta, double *P, cudaStream_t s)
{ if (nc) k_contact_out<<<GRID(nc)>>>(nc, vals, cij, gid, geo, cdel, Pa, Pb, nrm, delta, P); }
