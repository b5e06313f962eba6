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
// packed incidence of the canonical reduction (sweep_t2.cu): entries in 32-lane chunks, start[i]
// = packed position of particle i's list, wbase[g] = first packed entry of warp g's particles
extern thread_local bool g_t2_rows_by_contact;
extern thread_local bool g_t2_stage;
void to_planes(int64_t np, const double4 *in, double4 *out, cudaStream_t s);
extern thread_local int g_t2_exp;
struct PackedInc {
    const uint2 *inc;
    const uint32_t *start;
    const uint32_t *wbase;
    const G4 *geo;        // normals, rows of the stage: one copy per half-contact, packed order
    const R4 *row;
    const P8 *p8in;       // impulses of the sweep, one 32-byte slot per contact
    P8 *p8out;
};
void pack_rows(int64_t np, const uint2 *pinc, const G4 *geo, const R4 *row, G4 *gpk, R4 *rpk, cudaStream_t s);
void p8_pack(int64_t nc, const P4 *a, const P4 *b, P8 *o, cudaStream_t s);
void p8_unpack(int64_t nc, const P8 *q, P4 *a, P4 *b, cudaStream_t s);
void pack_plan(int64_t N, const uint32_t *inc_start, uint32_t *off_local, uint32_t *wsize, uint32_t *wbase,
               void *scan_tmp, cudaStream_t s, long long *launches);
void pack_fill(int64_t N, const uint32_t *inc_start, const uint2 *inc, const uint32_t *off_local, const uint32_t *wbase,
               uint32_t *pstart, uint2 *pinc, int64_t npacked, cudaStream_t s, long long *launches);
void launch_sweep(int mode, int64_t N, const uint32_t *order, const double4 *vin, const double4 *win, double4 *vout,
                  double4 *wout, const uint32_t *inc_start, const uint2 *inc, const PackedInc *pk, const G4 *geo,
                  const R4 *row,
                  const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out,
                  const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s);
bool sweep_uses_order();
void launch_tile_order(int64_t N, const uint32_t *inc_start, uint32_t *order, cudaStream_t s);
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
void launch_plate_hub(bool p8, int64_t n, const uint32_t *list, const uint2 *cij, const G4 *geo, const void *pin,
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
void set_sweep_variant(int v);      // 0 k_sweep_tile, 1 k_sweep_pipe, 2 k_sweep_ppt (bench/diagnostics)

// sweep5.cu: sweeps re-evaluating the contact geometry from positions (cb = SPOOK bias per contact)
enum { SWEEP5_PPT = 0, SWEEP5_PPT_PF = 1, SWEEP5_TILE = 2 };
void launch_sweep5(int kind, bool impact, int64_t N, const uint32_t *order, const double4 *pos, const double4 *vin,
                   const double4 *win, double4 *vout, double4 *wout, const uint32_t *inc_start, const uint2 *inc,
                   const double *cb, const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out,
                   const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s);
void launch_row_bias(int64_t nc, const R4 *row, double *cb, cudaStream_t s);
void launch_maxdiff(int64_t N, const double4 *a, const double4 *b, unsigned long long *out, cudaStream_t s);

// sweep_t2.cu: tile sweep with 256-bit records and conflict-free shared staging
void launch_sweep_t2(int64_t N, const double4 *vin, const double4 *win, double4 *vout, double4 *wout,
                     const uint32_t *inc_start, const uint2 *inc, const PackedInc *pk, const G4 *geo, const R4 *row,
                     const P4 *Pa_in, const P4 *Pb_in, P4 *Pa_out, P4 *Pb_out, const DevBoundary *bnd,
                     const SolveParams &sp, cudaStream_t s);
void run_sweep_t3(int variant, int n, int64_t N, int64_t nc, const double4 *vin, const double4 *win, double4 *vbuf[2],
                  double4 *wbuf[2], const uint32_t *inc_start, const uint2 *inc, const G4 *geo, const R4 *row,
                  P4 *Pa[2], P4 *Pb[2], void *scratch, const DevBoundary *bnd, const SolveParams &sp, cudaStream_t s,
                  double4 *vres, cudaEvent_t e0, cudaEvent_t e1);
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
