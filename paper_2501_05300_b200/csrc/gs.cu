// gs.cu -- coloured projected Gauss-Seidel ordering of the contact solve (the paper
// solves the MCP with PGS), the alternative to the Jacobi sweep k_sweep (sweep.cu).
//
// Colouring: two contacts conflict if they share a particle.  Priority pi(c) = SplitMix64 of the
// contact's public key (ties: smaller key first).  Jones-Plassmann rounds: an uncoloured contact
// all of whose higher-priority neighbours are coloured takes the smallest colour none of its
// coloured neighbours has.  A contact is coloured only after its higher-priority neighbours and
// before its lower-priority ones, so the result equals the sequential greedy colouring in
// decreasing priority that the oracle computes (oracle/dem_oracle.c or_color_contacts), and it
// does not depend on thread timing.
// Sweep: one launch per colour; the contacts of a colour touch disjoint particles, so each is
// updated from the latest velocities with the real inverse masses and applied at once, in place
// (no reduction, no atomics): one Gauss-Seidel sweep = the colours in increasing order.
#include "common.cuh"
#include "kernels.h"
#include "sweep_core.cuh"

__device__ __forceinline__ uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

// public key of a contact (canonical orientation: smaller gid first; walls/plates coded)
__device__ __forceinline__ uint64_t public_key(uint2 ij, const uint32_t *__restrict__ gid)
{
    const uint32_t gi = gid[ij.x];
    if (ij.y & PARTNER_EXT) {
        const uint32_t code = ij.y & ~PARTNER_EXT;
        const uint32_t kb = (code & PARTNER_PLATE) ? PLATE_KEY_BASE + 16u * ((code >> 4) & 0xF) + (code & 0xF)
                                                   : WALL_KEY_BASE + code;
        return ((uint64_t)gi << 32) | kb;
    }
    const uint32_t gj = gid[ij.y];
    return gj < gi ? (((uint64_t)gj << 32) | gi) : (((uint64_t)gi << 32) | gj);
}

__global__ void k_gs_init(int64_t nc, const uint2 *__restrict__ cij, const uint32_t *__restrict__ gid,
                          uint64_t *__restrict__ key, int *__restrict__ color)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    key[c] = public_key(cij[c], gid);
    color[c] = -1;
}

__device__ __forceinline__ bool higher(uint64_t ko, uint64_t kc)
{
    const uint64_t po = splitmix64(ko), pc = splitmix64(kc);
    return po > pc || (po == pc && ko < kc);
}

// one Jones-Plassmann round; newly coloured contacts counted in *n_new, > 256 colours in *fail
__global__ void k_gs_round(int64_t nc, const uint2 *__restrict__ cij, const uint32_t *__restrict__ inc_start,
                           const uint2 *__restrict__ inc, const uint64_t *__restrict__ key, int *color,
                           unsigned int *n_new, unsigned int *fail)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    volatile int *vcol = color;
    if (vcol[c] >= 0) return;
    const uint2 ij = cij[c];
    const uint64_t kc = key[c];
    uint32_t mask[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint32_t body[2] = {ij.x, ij.y};
    const int nb = (ij.y & PARTNER_EXT) ? 1 : 2;
    for (int q = 0; q < nb; q++) {
        const uint32_t s = inc_start[body[q]], e = inc_start[body[q] + 1];
        for (uint32_t k = s; k < e; k++) {
            const uint32_t o = inc[k].x & INC_CMASK;
            if (o == (uint32_t)c) continue;
            const int co = vcol[o];
            if (co < 0) {
                if (higher(key[o], kc)) return;            // wait for a higher-priority neighbour
            } else {
                mask[co >> 5] |= 1u << (co & 31);          // (only higher-priority ones can be coloured)
            }
        }
    }
    int col = -1;
    for (int w = 0; w < 8 && col < 0; w++)
        if (mask[w] != 0xffffffffu) col = 32 * w + __ffs(~mask[w]) - 1;
    if (col < 0) { atomicOr(fail, 1u); col = 255; }
    color[c] = col;
    atomicAdd(n_new, 1u);
}

__global__ void k_gs_sortkeys(int64_t nc, const int *__restrict__ color, uint64_t *__restrict__ keys,
                              uint32_t *__restrict__ vals, unsigned int *__restrict__ hist)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    keys[c] = ((uint64_t)color[c] << 32) | (uint64_t)c;
    vals[c] = (uint32_t)c;
    atomicAdd(&hist[color[c]], 1u);
}

// one colour: every contact of the colour updated from the latest velocities, applied in place
__global__ void k_gs_color(uint32_t n, const uint32_t *__restrict__ ord, const uint2 *__restrict__ cij,
                           const G4 *__restrict__ geo, const R4 *__restrict__ row, P4 *Pa, P4 *Pb, double4 *vel,
                           double4 *ang, const uint32_t *__restrict__ inc_start, const DevBoundary *__restrict__ bnd,
                           SolveParams sp)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint32_t c = ord ? ord[t] : t;      // ord == nullptr: the arrays are already in colour order
    const uint2 ij = cij[c];
    const uint32_t a = ij.x, p = ij.y;
    // real inverse masses: the stored weights are c/m, c/I (mass splitting) -> divide by c
    const double4 VA0 = vel[a], WA0 = ang[a];
    const double ca = (double)(inc_start[a + 1] - inc_start[a]);
    const double4 VA = make_double4(VA0.x, VA0.y, VA0.z, VA0.w / ca), WA = make_double4(WA0.x, WA0.y, WA0.z, WA0.w / ca);
    double4 VB, WB, VB0, WB0;
    double mt = sp.mu_t, cbn = 1.0;
    const bool ext = (p & PARTNER_EXT) != 0;
    if (!ext) {
        VB0 = vel[p];
        WB0 = ang[p];
        cbn = (double)(inc_start[p + 1] - inc_start[p]);
        VB = make_double4(VB0.x, VB0.y, VB0.z, VB0.w / cbn);
        WB = make_double4(WB0.x, WB0.y, WB0.z, WB0.w / cbn);
    } else {
        d3 bv;
        double mr;
        boundary_body(p, bnd, bv, mt, mr);
        VB = make_double4(bv.x, bv.y, bv.z, 0.0);
        WB = make_double4(0.0, 0.0, 0.0, 0.0);
    }
    const G4 g = geo[c];
    const R4 rw = row[c];
    const ContactOut r = contact_core(VA, WA, VB, WB, mt, mk(g.x, g.y, g.z), g.w, rw.x, rw.y, rw.z, rw.w, Pa[c], Pb[c],
                                      sp.rolling_dims);
    Pa[c] = r.Pa;
    Pb[c] = r.Pb;
    const double la = rw.z, lb = rw.w;
    double4 V = VA0, W = WA0;
    V.x -= VA.w * r.L.x; V.y -= VA.w * r.L.y; V.z -= VA.w * r.L.z;
    W.x -= WA.w * (la * r.nxdPt.x + r.dPr.x); W.y -= WA.w * (la * r.nxdPt.y + r.dPr.y);
    W.z -= WA.w * (la * r.nxdPt.z + r.dPr.z);
    vel[a] = V;
    ang[a] = W;
    if (!ext) {
        V = VB0;
        W = WB0;
        V.x += VB.w * r.L.x; V.y += VB.w * r.L.y; V.z += VB.w * r.L.z;
        W.x += WB.w * (-lb * r.nxdPt.x + r.dPr.x); W.y += WB.w * (-lb * r.nxdPt.y + r.dPr.y);
        W.z += WB.w * (-lb * r.nxdPt.z + r.dPr.z);
        vel[p] = V;
        ang[p] = W;
    }
}

// ------------------------------------------------------------------ host side
// colours the contacts; ord = contacts sorted by colour, cstart[0..ncol] colour ranges (host)
int gs_color(int64_t nc, const uint2 *cij, const uint32_t *gid, const uint32_t *inc_start, const uint2 *inc,
             uint64_t *key, int *color, uint64_t *keys[2], uint32_t *vals[2], void *sort_tmp, unsigned int *dscr,
             std::vector<uint32_t> &cstart, cudaStream_t s, long long *launches)
{
    cstart.assign(1, 0);
    if (!nc) return 0;
    const unsigned gb = (unsigned)((nc + 255) / 256);
    k_gs_init<<<gb, 256, 0, s>>>(nc, cij, gid, key, color);
    unsigned int h[2] = {0, 0};
    int64_t done = 0;
    for (int round = 0; round < 100000 && done < nc; round++) {
        cudaMemsetAsync(dscr, 0, 2 * sizeof(unsigned int), s);
        k_gs_round<<<gb, 256, 0, s>>>(nc, cij, inc_start, inc, key, color, dscr, dscr + 1);
        cudaMemcpyAsync(h, dscr, 2 * sizeof(unsigned int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (h[1]) return -1;
        done += h[0];
        *launches += 1;
    }
    unsigned int *hist = dscr + 2;
    cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned int), s);
    k_gs_sortkeys<<<gb, 256, 0, s>>>(nc, color, keys[0], vals[0], hist);
    radix_sort_u64(keys, vals, nc, 40, sort_tmp, s, launches);
    unsigned int hh[256];
    cudaMemcpyAsync(hh, hist, sizeof(hh), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    int ncol = 0;
    for (int q = 0; q < 256; q++)
        if (hh[q]) ncol = q + 1;
    for (int q = 0; q < ncol; q++) cstart.push_back(cstart.back() + hh[q]);
    *launches += 2;
    return ncol;
}

void gs_sweep(const std::vector<uint32_t> &cstart, const uint32_t *ord, const uint2 *cij, const G4 *geo, const R4 *row,
              P4 *Pa, P4 *Pb, double4 *vel, double4 *ang, const uint32_t *inc_start, const DevBoundary *bnd,
              const SolveParams &sp, cudaStream_t s, long long *launches)
{
    for (size_t q = 0; q + 1 < cstart.size(); q++) {
        const uint32_t n = cstart[q + 1] - cstart[q], o = cstart[q];
        if (!n) continue;
        if (ord)
            k_gs_color<<<(n + 127) / 128, 128, 0, s>>>(n, ord + o, cij, geo, row, Pa, Pb, vel, ang, inc_start, bnd, sp);
        else   // colour-ordered records: each colour reads a contiguous, coalesced range
            k_gs_color<<<(n + 127) / 128, 128, 0, s>>>(n, nullptr, cij + o, geo + o, row + o, Pa + o, Pb + o, vel, ang,
                                                       inc_start, bnd, sp);
        *launches += 1;
    }
}

// contact records into colour order (once per step and stage) and the impulses back
__global__ void k_gs_gather(int64_t nc, const uint32_t *__restrict__ ord, const uint2 *__restrict__ cij,
                            const G4 *__restrict__ geo, const R4 *__restrict__ row, const P4 *__restrict__ Pa,
                            const P4 *__restrict__ Pb, uint2 *__restrict__ cijO, G4 *__restrict__ geoO,
                            R4 *__restrict__ rowO, P4 *__restrict__ PaO, P4 *__restrict__ PbO)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nc) return;
    const uint32_t c = ord[t];
    if (cijO) cijO[t] = cij[c];
    if (geoO) geoO[t] = geo[c];
    if (rowO) rowO[t] = row[c];
    if (PaO) { PaO[t] = Pa ? Pa[c] : mkP4(0, 0, 0, 0); PbO[t] = Pb ? Pb[c] : mkP4(0, 0, 0, 0); }
}
__global__ void k_gs_scatter(int64_t nc, const uint32_t *__restrict__ ord, const P4 *__restrict__ PaO,
                             const P4 *__restrict__ PbO, P4 *__restrict__ Pa, P4 *__restrict__ Pb)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nc) return;
    const uint32_t c = ord[t];
    Pa[c] = PaO[t];
    Pb[c] = PbO[t];
}
void gs_gather(int64_t nc, const uint32_t *ord, const uint2 *cij, const G4 *geo, const R4 *row, const P4 *Pa,
               const P4 *Pb, uint2 *cijO, G4 *geoO, R4 *rowO, P4 *PaO, P4 *PbO, cudaStream_t s)
{ if (nc) k_gs_gather<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, ord, cij, geo, row, Pa, Pb, cijO, geoO, rowO, PaO, PbO); }
void gs_scatter(int64_t nc, const uint32_t *ord, const P4 *PaO, const P4 *PbO, P4 *Pa, P4 *Pb, cudaStream_t s)
{ if (nc) k_gs_scatter<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, ord, PaO, PbO, Pa, Pb); }
