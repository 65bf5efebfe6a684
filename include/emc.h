/* emc.h -- C ABI of libemc.so, the B200 (sm_100a) event-based Monte Carlo
 * transport engine.  Plain pointers and sizes only; no torch types.
 *
 * Every entry point replaces one compiled-kernel call of the reference
 * package eventmc (/root/reference/pkg/src/eventmc); the reference's Python
 * layer reaches those kernels through numba dispatch, so the "FFI" this ABI
 * stands in for is the argument tuple of each @njit function.  The binding a
 * maintainer adds on the reference side is shown in INTEGRATION.md.
 *
 * Ownership: the context owns every device buffer (library, geometry,
 * particle slots, queues, fission bank, contribution log); callers own host
 * buffers and pass them in/out.  All calls are synchronous w.r.t. the host
 * unless stated, run on the stream set by emc_set_stream (default: the
 * legacy stream), and return 0 on success or a negative EMC_E_* code; the
 * message is in emc_last_error().  Transport errors detected on the device use
 * the reference's codes (kernels.py:108-113) in emc_batch_result.error.
 */
#ifndef EMC_H
#define EMC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMC_ABI_VERSION 2   /* 2: box_guard in emc_run_config; grid index, union backends, groups */
#define EMC_N_COUNTERS 24   /* kernels.py:81-103 layout */
#define EMC_N_TIMINGS 4     /* kernels.py:115-120: lookup, advance, collision, sort */

enum {
    EMC_OK = 0,
    EMC_E_CUDA = -1,       /* CUDA runtime failure */
    EMC_E_ARG = -2,        /* invalid argument / call order */
    EMC_E_OOM = -3,        /* device allocation failed */
    EMC_E_RANGE = -4       /* problem exceeds an encoding limit */
};

/* Box guard (extension, off by default = the reference): the reference's
 * reflect-and-nudge (kernels.py:782-797) and its DIST_EPS skip (K:418-492) can
 * leave a particle just outside the reflective box; a fission site banked there
 * stops the next batch with EMC_ERR_OUTSIDE_BOX (K:989-992).  With box_guard = 1
 * a particle found outside the box after a move is put back on the box face it
 * passed with that direction component pointing inward (vacuum geometry: it
 * leaks).  Histories that stay inside are untouched, bit for bit; the number of
 * guarded moves is counter EMC_CNT_BOX_GUARD. */
#define EMC_CNT_BOX_GUARD 23

/* transport error codes (kernels.py:108-113) */
enum { EMC_ERR_NO_SURFACE = 1, EMC_ERR_OUTSIDE_BOX = 2, EMC_ERR_STREAM_OVERLAP = 3,
       EMC_ERR_RUNAWAY_HISTORY = 4, EMC_ERR_QUEUE_STATE = 5, EMC_ERR_NONPOSITIVE_SIGMA = 6 };

typedef struct emc_ctx emc_ctx;

/* Library.arrays() (xslib.py:119-153): nuclide grids + channels, material
 * compositions, global energy bounds. */
typedef struct {
    int64_t n_nuclides, n_points, n_materials, n_entries;
    const int64_t *grid_off;                 /* [n_nuclides+1] */
    const double *grids, *ch_t, *ch_s, *ch_c, *ch_f; /* [n_points] */
    const double *nu;                        /* [n_nuclides] */
    const int64_t *mat_off;                  /* [n_materials+1] */
    const int32_t *mat_nuc;                  /* [n_entries] */
    const double *mat_den;                   /* [n_entries] */
    double emin, emax;
} emc_library;

/* Pincell.as_tuple() (geometry.py:83-90) */
typedef struct {
    double radius, r2, half_pitch, height;
    int64_t n_axial;
    const double *zplanes;                   /* [n_axial+1] */
    const int32_t *fuel_mats;                /* [n_axial] */
    int64_t mod_mat;
} emc_geometry;

/* RunConfig (transport.py:26-99) restricted to what the engine consumes, plus
 * this rank's contiguous block of particle indices [gid_lo, gid_lo+n_assigned). */
typedef struct {
    int64_t particles_per_batch;             /* pmax in the stream layout */
    int64_t gid_lo, n_assigned;
    int64_t max_in_flight;
    int32_t history;                         /* 1: history-based executor */
    int32_t fused;                           /* tally_mode == "fused" */
    int32_t use_logs;                        /* reduction == "deterministic" */
    int32_t sort_enabled, sort_every;
    int32_t box_guard;                       /* extension (RunConfig.box_guard), 0 = the reference */
    uint64_t seed;
    double alpha, fission_t;
    int64_t perturb_gid;                     /* -1: none */
} emc_run_config;

typedef struct {
    int64_t batch;
    double k_run;
    int32_t batch0, score;                   /* score = active batch */
} emc_batch_args;

typedef struct {
    int64_t counters[EMC_N_COUNTERS];
    double timings[EMC_N_TIMINGS];           /* seconds, CUDA events */
    int64_t n_sites, n_logs, iterations, launches;
    int32_t error;                           /* EMC_ERR_* or 0 */
    int32_t reruns;                          /* overflow grow-and-rerun count (R:122-142) */
    int64_t error_gid;
} emc_batch_result;

const char *emc_last_error(void);
int emc_abi_version(void);
int emc_device_count(int *n);

int emc_create(int device, emc_ctx **out);
void emc_destroy(emc_ctx *ctx);
/* use an existing cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) */
int emc_set_stream(emc_ctx *ctx, void *cuda_stream);

/* replaces the lib tuple built at replication.py:169 */
int emc_upload_library(emc_ctx *ctx, const emc_library *lib);
/* replaces the geom tuple built at replication.py:171 */
int emc_upload_geometry(emc_ctx *ctx, const emc_geometry *geom);
/* Extensions beyond the reference (fixed-source shielding
 * slab with 3D mesh flux tallies; parity pinned against the oracle's
 * restatement of the same extension, not against the reference):
 *   slab = 1: no fuel cylinder, the box is n_axial material layers in z;
 *   vacuum = 1: outer box planes leak (counter 22) instead of reflecting;
 *   fixed source: every batch samples a surface source on z = 0 (energy, or
 *   the fission spectrum when energy == 0) instead of resampling a bank;
 *   mesh: nx*ny*nz track-length (flux, total rate) tally over the box, one
 *   batch's sums at emc_mesh_device() after each emc_run_batch (2 per cell). */
int emc_set_geometry_options(emc_ctx *ctx, int32_t slab, int32_t vacuum);
/* Lattice extension (BASELINE config 2): n x n pin cells of
 * `pitch` filling the box (emc_geometry.half_pitch must be n*pitch/2);
 * pin_map[j*n+i] != 0: fuel pin of `radius` with the axial fuel materials,
 * 0: water hole.  Batch 0 samples a fuel pin uniformly, then its disk.
 * n <= 1 restores the reference's single pincell. */
int emc_set_lattice(emc_ctx *ctx, int32_t n, double pitch, const int32_t *pin_map);
int emc_set_fixed_source(emc_ctx *ctx, int32_t enabled, double energy);
int emc_set_mesh(emc_ctx *ctx, int32_t nx, int32_t ny, int32_t nz);
int emc_mesh_device(emc_ctx *ctx, double **ptr, int64_t *n);

/* replaces _Worker allocation (replication.py:62-111) */
int emc_configure(emc_ctx *ctx, const emc_run_config *cfg);

/* source of batch b>0: systematic resampling (transport.py:188-200) with
 * uniform u of the canonical bank of batch b-1 -- either this context's own
 * bank (single rank) or a device-resident global bank (multi-rank, 7 arrays
 * x,y,z,dx,dy,dz,E of length n that stay valid during the next batch) */
int emc_set_source_local(emc_ctx *ctx, double u);
int emc_set_source_device(emc_ctx *ctx, const void *const ptrs[7], int64_t n, double u);
/* same, when the arrays hold only the window of the global bank this rank
 * resamples from: element j is global site (lo + j) mod n (multi-GPU bank
 * exchange, replaces the R:221-228 gather + R:271-280 resample for a rank) */
int emc_set_source_window(emc_ctx *ctx, const void *const ptrs[7], int64_t n, double u, int64_t lo);

/* one worker-batch: replaces kernels.run_event_batch / run_history_batch
 * (kernels.py:1043-1211) as called at replication.py:127-138, including the
 * grow-and-rerun on buffer overflow.  Leaves the canonical (parent, ordinal)
 * sorted fission bank of this rank on the device. */
int emc_run_batch(emc_ctx *ctx, const emc_batch_args *args, emc_batch_result *res);

/* batch sums of this rank (tally.py:66-93): deterministic mode folds the
 * contribution log in canonical order starting from init (NULL = zeros; a
 * previous rank's partial sums to chain ranks bit-exactly); fast mode returns
 * the atomically accumulated bins (+init). */
int emc_reduce_bins(emc_ctx *ctx, const double *init, double *out, int64_t n_bins);

/* canonical bank of the last batch */
int emc_bank_size(emc_ctx *ctx, int64_t *n);
int emc_bank_device(emc_ctx *ctx, void *ptrs[9]);  /* parent,ord,x,y,z,dx,dy,dz,E */
int emc_bank_copy(emc_ctx *ctx, int64_t start, int64_t n, int64_t *parent, int32_t *ord,
                  double *x, double *y, double *z, double *dx, double *dy, double *dz,
                  double *E);

/* --- single-operation entry points (public API wrappers) --- */
/* Union-grid lookup backends (RunConfig.accel != "binary"; replication.py
 * _union_for R:145-152 -> xslib.union_tuple X:166-172): the union energy grid
 * ugrid[n] (strictly ascending), the bracket map map[n][n_nuclides]
 * (build_unionized_index, X:321-339) and, for "unionized", the merged bounding
 * channels merged[n][n_nuclides][8] (merge_channels X:342-358; nullable).
 * Replaced by the next library upload. */
int emc_upload_union(emc_ctx *ctx, const double *ugrid, int64_t n, const int32_t *map, const double *merged);
/* lookup backend of transport and emc_xs_lookup: 0 binary (the device's
 * log-hash + scan, bit-identical to the binary search), 1 double_index,
 * 2 unionized (kernels.py ACCEL_* codes; K:306-320) */
int emc_set_accel(emc_ctx *ctx, int32_t accel);
/* Single-process multi-GPU group (SURVEY 8b's init-over-devices, bank
 * exchange and bin all-reduce entries; replication.py:155-286 with W
 * workers): ranks = contexts configured for the contiguous particle blocks
 * [r*P/W, (r+1)*P/W), one per GPU (a GPU may hold several, e.g. for tests).
 * After every rank's emc_run_batch:
 *   emc_group_reduce_bins(g, out, n_bins): tallies over the ranks --
 *     deterministic: chained fold, bit-identical to one rank; fast: rank-ordered
 *     sum of the rank bins (R:238-240);
 *   emc_group_exchange_bank(g, ppb, u, &n): every rank's resampling window of
 *     the global canonical bank (rank-ordered concatenation, R:221-228) copied
 *     device to device (peer copies) and installed as its source (replaces
 *     emc_set_source_local, R:271-280); n = global bank size. */
typedef struct emc_group emc_group;
int emc_group_create(emc_ctx *const *ctxs, int32_t n, emc_group **out);
void emc_group_destroy(emc_group *g);
int emc_group_reduce_bins(emc_group *g, double *out, int64_t n_bins);
int emc_group_exchange_bank(emc_group *g, int64_t ppb, double u, int64_t *out_n);

/* kernels.macro_lookup_full (kernels.py:287-331): sums[n][5], partials[n][max_comp][4] (nullable) */
int emc_xs_lookup(emc_ctx *ctx, int64_t n, const int32_t *mats, const double *E, double *sums,
                  double *partials, int32_t max_comp);
/* grid search of one composition entry (material entry k of mat_nuc, i.e. one
 * nuclide's grid) at energy E, by the device's log-hash + forward scan
 * (emc_device.cuh: bracket).  out[n][2] = (state, i): state 0 interior with
 * grid[i] <= E < grid[i+1] (searchsorted(grid, E, 'right') - 1), 1 clamp to the
 * first point (E <= grid[0], i = 0), 2 clamp to the last (E >= grid[-1],
 * i = len-1) -- the reference's K:600-621 cases.  Parity hook for the grid
 * indices north_star requires bit-exact. */
int emc_grid_index(emc_ctx *ctx, int64_t n, const int32_t *entry, const double *E, int32_t *out);
/* kernels.locate_point (kernels.py:403-415): out[n][3] = kind, axial, material */
int emc_locate(emc_ctx *ctx, int64_t n, const double *pos, int32_t *out);
/* kernels.boundary_distance (kernels.py:418-492): cell[n][2] = kind, axial */
int emc_distance(emc_ctx *ctx, int64_t n, const double *pos, const double *dir,
                 const int32_t *cell, double *dist, int32_t *surf);
/* transport.sample_isotropic / sample_collision_distance (transport.py:161-174) */
int emc_particle_ops(emc_ctx *ctx, int64_t n, const uint64_t *states, const double *sigma_t,
                     double *iso, double *dcol, uint64_t *state_iso, uint64_t *state_dcol);
/* kernels.sort_queue (kernels.py:1014-1035): stable sort of q by (mat[q], E[q]) */
int emc_sort_queue(emc_ctx *ctx, int64_t n, const int32_t *q, int64_t n_slots,
                   const int32_t *mat, const double *E, int32_t *out);
/* kernels.replay_into_bins (kernels.py:1219-1223): sums[b] += vals in order */
int emc_replay_bins(emc_ctx *ctx, int64_t n, const int32_t *bin, const double *val,
                    int32_t n_bins, double *sums);
/* kernels.lcg_skip (kernels.py:144-158) */
int emc_lcg_skip(emc_ctx *ctx, int64_t n, const uint64_t *state, const uint64_t *k, uint64_t *out);
/* device log/sin/cos replicas (emc_libm.h): out[n][3] */
int emc_libm_eval(emc_ctx *ctx, int64_t n, const double *x, double *out);

/* division used by the staged lookup (precomputed reciprocal + one FMA
 * correction) next to the IEEE division: out[2i] = staged n/d, out[2i+1] =
 * n/d correctly rounded; they must be equal bit for bit (parity test) */
int emc_div_eval(emc_ctx *ctx, int64_t n, const double *num, const double *den, double *out);

/* tuning harness: mean ms of a lookup kernel over n (material, energy)
 * pairs: variant 8 = the shared-memory-staged production lookup, any other
 * value = the plain gather lookup (macro_tcf) it replaced */
int emc_bench_lookup(emc_ctx *ctx, int64_t n, const int32_t *mats, const double *E, int32_t variant,
                     int32_t iters, double *ms, double *checksum);

/* number of kernel launches issued by this context so far */
int64_t emc_launch_count(emc_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* EMC_H */
