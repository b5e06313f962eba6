// kernels.h -- host launchers of the device kernels (detect.cu, solve.cu); internal to libdem.so.
#pragma once
#include <string>
#include <vector>

#include "../../include/dem.h"
#include "common.cuh"

// detect.cu
void launch_keys(int64_t N, const double4 *pos, const GridParams &g, uint64_t *keys, uint32_t *vals, cudaStream_t s);
void launch_permute(int64_t N, const uint32_t *idx, const double4 *pin, const double4 *vin, const double4 *win,
                    const uint32_t *gin, double4 *pout, double4 *vout, double4 *wout, uint32_t *gout, cudaStream_t s);
void launch_cells(int64_t N, const uint64_t *keys, const GridParams &g, uint32_t *cs, uint32_t *ce, cudaStream_t s);
void launch_broad(bool fill, int64_t N, const double4 *pos, const GridParams &g, const uint32_t *cs,
                  const uint32_t *ce, const DevBoundary *bnd, uint32_t *cnt_or_start, uint2 *cand, cudaStream_t s);
void launch_trans(int64_t N, int64_t nc, const uint2 *cand, uint32_t *cnt, uint32_t *ct_start, uint32_t *cursor,
                  uint32_t *ct_list, void *scan_tmp, cudaStream_t s, long long *launches);
void launch_hist_flag(int64_t nc, const P4 *Pa, const P4 *Pb, uint32_t *flag, cudaStream_t s);
void launch_hist_keys(int64_t nc, const uint32_t *flag, const uint32_t *scan, const uint2 *cand, const uint32_t *gid,
                      uint64_t *keys, uint32_t *vals, cudaStream_t s);
void launch_hist_gather(int64_t nh, const uint32_t *vals, const uint2 *cand, const uint32_t *gid, const P4 *Pa,
                        const P4 *Pb, P4 *hPa, P4 *hPb, cudaStream_t s);
void launch_hist_carry(int64_t nc, const uint2 *cand, const uint32_t *gid, const uint64_t *hkey, const P4 *hPa,
                       const P4 *hPb, int64_t nh, P4 *Pa, P4 *Pb, cudaStream_t s);
void launch_narrow(int64_t nc, const uint2 *cand, const double4 *pos, const DevBoundary *bnd, uint32_t *flag,
                   P4 *Pa, P4 *Pb, StepScalars *sc, cudaStream_t s);
void launch_compact(int64_t nc, const uint2 *cand, const uint32_t *flag, const uint32_t *scan, const double4 *pos,
                    const DevBoundary *bnd, const SolveParams &sp, const P4 *Pca, const P4 *Pcb, uint2 *cij,
                    G4 *geo, R4 *row, double *cdel, P4 *Pa, P4 *Pb, uint32_t *ccand, const uint32_t *gid, StepScalars *sc,
                    cudaStream_t s);
void launch_count_kinds(int64_t nc, const uint8_t *own, const uint2 *cij, const uint32_t *gid, StepScalars *sc, cudaStream_t s);
void launch_inc(int64_t N, const uint32_t *co_start, const uint2 *cand, const uint32_t *scan, const uint32_t *ct_start,
                const uint32_t *ct_list, const uint32_t *flag, const uint32_t *gid, uint32_t *cnt, uint32_t *inc_start,
                uint2 *inc, void *scan_tmp, cudaStream_t s, long long *launches);
void launch_contact_keys(int64_t nc, const uint8_t *own, const uint2 *cij, const uint32_t *gid, uint64_t *keys, uint32_t *vals,
                         unsigned int *cnt, cudaStream_t s);
void launch_contact_out(int64_t nc, const uint32_t *vals, const uint2 *cij, const uint32_t *gid, const G4 *geo,
                        const double *cdel, const P4 *Pa, const P4 *Pb, double *nrm, double *delta, double *P, cudaStream_t s);

// solve.cu
enum { SWEEP_MODE_SWEEP = 0, SWEEP_MODE_APPLY = 1, SWEEP_MODE_FORCES = 2 };
void launch_prepare(int64_t N, const uint32_t *inc_start, const double4 *pos, double4 *vel, double4 *ang, double rho,
                    cudaStream_t s);
void launch_rows(int64_t nc, int mode, const uint2 *cij, const G4 *geo, const double *cdel, R4 *row, R4 *row_imp,
                 const double4 *vel, const double4 *pos, const DevBoundary *bnd, const SolveParams &sp, StepScalars *sc,
                 cudaStream_t s);
void launch_apply(int mode, int64_t N, const double4 *vin, const double4 *win, double4 *vout, double4 *wout,
                  const uint32_t *inc_start, const uint2 *inc, const G4 *geo, const R4 *row, const P4 *Pa,
                  const P4 *Pb, const SolveParams &sp, cudaStream_t s);
void launch_integrate(int64_t N, const uint8_t *own, double4 *pos, const double4 *vel, const double4 *ang, const double4 *xref, double h,
                      double rho, double *ke_part, StepScalars *sc, cudaStream_t s);
void launch_plate_sum(int64_t nc, const uint8_t *own, const uint2 *cij, const G4 *geo, const P4 *Pa, unsigned long long *acc,
                      unsigned int *pcount, cudaStream_t s);
void launch_boundary(DevBoundary *bnd, const unsigned long long *acc, const unsigned int *pcount, double h, StepScalars *sc,
                     cudaStream_t s);
// dist.cu: history hand-over at rebuilds (HistRec = 48 bytes: key, pad, P_a, P_b)
constexpr size_t HIST_REC_BYTES = 48;
void launch_hist_auth(int64_t nh, const uint32_t *vals, const uint2 *cand, const uint8_t *own, uint8_t *auth, cudaStream_t s);
void launch_gid_list(int64_t n, const uint32_t *idx, const uint32_t *gid, uint64_t *out, cudaStream_t s);
void launch_hist_select(int64_t nh, const uint64_t *hkey, const uint8_t *auth, const uint64_t *B, int64_t nB, uint32_t *flag,
                        cudaStream_t s);
void launch_hist_pack(int64_t n, const uint32_t *idx, const uint64_t *hkey, const P4 *hPa, const P4 *hPb, void *out,
                      cudaStream_t s);
void launch_hist_unpack(int64_t n, const void *in, uint64_t *key, uint32_t *val, uint32_t val0, P4 *Pa, P4 *Pb,
                        cudaStream_t s);
void launch_iota_keys(int64_t n, const uint64_t *hkey, uint64_t *key, uint32_t *val, cudaStream_t s);
void launch_hist_last(int64_t n, const uint64_t *key, uint32_t *flag, cudaStream_t s);
void launch_hist_emit(int64_t n, const uint32_t *flag, const uint32_t *scan, const uint64_t *key, const uint32_t *val,
                      const P4 *Pa, const P4 *Pb, uint64_t *okey, P4 *oPa, P4 *oPb, cudaStream_t s);
void launch_hist_x(int64_t n, const uint8_t *own, const double4 *pos, double lo, double hi, int nb,
                   unsigned long long *hist, cudaStream_t s);
void launch_first_bad(int64_t nc, int64_t N, const uint8_t *own, const uint2 *cij, const uint32_t *gid, const P4 *Pa,
                      const P4 *Pb, const double4 *pos, const double4 *vel, const double4 *ang,
                      unsigned long long *out, cudaStream_t s);
void launch_plate_list_flags(int64_t nc, const uint8_t *own, const uint2 *cij, uint32_t *flag, cudaStream_t s);
void launch_plate_hub(int64_t n, const uint32_t *list, const uint2 *cij, const G4 *geo, const void *pin,
                      const void *pout, unsigned long long *acc, cudaStream_t s);
void launch_plate_kick(DevBoundary *bnd, unsigned long long *acc, double h, int first, cudaStream_t s);
void launch_keep(int64_t n, const double *x, int axis, double lo, double hi, uint32_t *flag, cudaStream_t s);
void launch_keep_gather(int64_t n, const uint32_t *flag, const uint32_t *scan, const double *x, const double *r,
                        const double *v, const double *w, const uint32_t *g, double *ox, double *orr, double *ov,
                        double *ow, uint32_t *og, cudaStream_t s);
void launch_residuals(int64_t nc, const uint8_t *own, const uint2 *cij, const G4 *geo, const R4 *row, const double4 *vel,
                      const P4 *Pa, const P4 *Pb, const DevBoundary *bnd, const SolveParams &sp, StepScalars *sc,
                      cudaStream_t s);
void launch_scatter_P(int64_t nc, const uint32_t *ccand, const P4 *Pa, const P4 *Pb, P4 *Pca, P4 *Pcb,
                      cudaStream_t s);
void launch_to_gid_order(int64_t N, int64_t n_sorted, const uint8_t *own, const uint32_t *gid, const uint32_t *gid_sorted, const double4 *a,
                         const double4 *b, const double4 *c, double *oa, double *ob, double *oc, double *orad,
                         uint32_t *ogid, cudaStream_t s);
void launch_load_state(int64_t N, const double *x, const double *r, const double *v, const double *w,
                       const uint32_t *gid_in, double4 *pos, double4 *vel, double4 *ang, uint32_t *gid, cudaStream_t s);
// sweep.cu: the contact-once tile sweep.  Tiles of SWEEP_TILE particles; items =
// contacts owned by a tile (intra-tile pairs once, cross-tile pairs once per side, boundary
// contacts once); item meta word: flags + partner (see IT_*).
#ifndef SWEEP_TILE
#define SWEEP_TILE 256           // <= 512: the owner index is 9 bits
#endif
#ifndef SWEEP_SLOT_CAP
#define SWEEP_SLOT_CAP (3 * SWEEP_TILE)
#endif
#ifndef SWEEP_MINB
#define SWEEP_MINB 2
#endif
#ifndef SWEEP_SIG16
#define SWEEP_SIG16 0            // 1: scale exponents as int16 pairs and bad flags as a bitmask (-4 KB of shared memory per CTA)
#endif
#ifndef SWEEP_TMA
#define SWEEP_TMA 1              // tile staging by TMA bulk copies on an mbarrier (0: per-thread cp.async)
#endif
#define IT_INTRA 0x80000000u     // partner in the tile, body b's share goes to slot (bits 9..20)
#define IT_B 0x40000000u         // cross pair: the owner is the canonical body b
#define IT_EXT 0x20000000u       // wall / plate box: bits 0..28 = boundary code (PARTNER_* codes)
#define IT_IDX 0x1FFFFFFFu       // cross pair: partner's local index (< 2^29)
#define IT_LOC 0x1FFu            // intra pair: partner's index in the tile
#define IT_SLOT_SHIFT 9
#define IT_SLOT_MASK 0xFFFu
struct __align__(32) CRec { double nx, ny, nz, delta; };  // per item, per stage (meta in n's low bits, sweep.cu)
struct __align__(32) PRec { double pn, pt[3], pr[3], b; }; // per item, ping-pong: fp64 impulses + SPOOK bias
static_assert(sizeof(CRec) == 32 && sizeof(PRec) == 64, "item records");
struct SweepPlan {
    uint32_t *istart = nullptr;   // [N+1] first item of each particle (tile-contiguous)
    uint32_t *pin = nullptr;      // [N] slot range in the tile: start | count << 16
    uint8_t *noint = nullptr;     // [tiles] 1: the tile's intra pairs are evaluated as cross pairs
    uint32_t *slot_of = nullptr;  // [nc] slot of an intra contact at body b
    uint32_t *item_c = nullptr;   // [items] contact index
    uint32_t *item_meta = nullptr;// [items] meta word
    uint16_t *item_own = nullptr; // [items] owner's index in the tile
    uint32_t *wrange = nullptr;   // [tiles * (TT/32 + 1)] the sweep warps' item ranges
    double *rad = nullptr;        // [N] radius
};
void plan_counts(int64_t N, const uint32_t *inc_start, const uint2 *inc, const SweepPlan &pl, uint32_t *nitem,
                 uint32_t *nin, unsigned int *any_full, void *scan_tmp, cudaStream_t s, long long *launches);
void plan_fill(int64_t N, const uint32_t *inc_start, const uint2 *inc, const double4 *pos, const SweepPlan &pl,
               cudaStream_t s, long long *launches);
void item_pack(int64_t n, const SweepPlan &pl, const G4 *geo, const double *cdel, const R4 *row, const P4 *Pa,
               const P4 *Pb, CRec *rec, PRec *P, cudaStream_t s);
void item_unpack(int64_t n, const SweepPlan &pl, const CRec *rec, const PRec *P, P4 *Pa, P4 *Pb, cudaStream_t s);
void launch_sweep_items(bool impact, int64_t N, const double4 *vin, const double4 *win, const double *rad, double4 *vout,
                        double4 *wout, const SweepPlan &pl, const CRec *rec, const PRec *Pin, PRec *Pout,
                        const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s);
void launch_plate_items_flag(int64_t n, const uint8_t *own, const SweepPlan &pl, const uint2 *cij, uint32_t *flag,
                             cudaStream_t s);
void launch_plate_hub_items(int64_t n, const uint32_t *list, const SweepPlan &pl, const G4 *geo, const CRec *rec,
                            const PRec *pin, const PRec *pout, unsigned long long *acc, cudaStream_t s);
// generate.cu: on-device bed generator (include/dem.h dem_generator)
bool generate_bed(const dem_generator &g, const dem_box &box, double slab_lo, double slab_hi,
                  void *(*alloc)(size_t, void *), void *actx, cudaStream_t s, double **x, double **r, uint32_t **gid,
                  int64_t *n, std::string &err);
// gs.cu: coloured Gauss-Seidel ordering
int gs_color(int64_t nc, const uint2 *cij, const uint32_t *gid, const uint32_t *inc_start, const uint2 *inc,
             uint64_t *key, int *color, uint64_t *keys[2], uint32_t *vals[2], void *sort_tmp, unsigned int *dscr,
             std::vector<uint32_t> &cstart, cudaStream_t s, long long *launches);
void gs_gather(int64_t nc, const uint32_t *ord, const uint2 *cij, const G4 *geo, const R4 *row, const P4 *Pa,
               const P4 *Pb, uint2 *cijO, G4 *geoO, R4 *rowO, P4 *PaO, P4 *PbO, cudaStream_t s);
void gs_scatter(int64_t nc, const uint32_t *ord, const P4 *PaO, const P4 *PbO, P4 *Pa, P4 *Pb, cudaStream_t s);
void gs_sweep(const std::vector<uint32_t> &cstart, const uint32_t *ord, const uint2 *cij, const G4 *geo, const R4 *row,
              P4 *Pa, P4 *Pb, double4 *vel, double4 *ang, const uint32_t *inc_start, const DevBoundary *bnd,
              const SolveParams &sp, cudaStream_t s, long long *launches);
