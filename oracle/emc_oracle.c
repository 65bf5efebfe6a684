/* CPU ORACLE -- test infrastructure only.
 *
 * A plain-C restatement of the reference transport kernels
 * (/root/reference/pkg/src/eventmc/kernels.py, cited below as K:<line>),
 * used ONLY as the parity checker by tests/, by __graft_entry__.smoke() and
 * as the CPU baseline leg of bench.py.  The product path (libemc.so, CUDA)
 * never links or calls this file.
 *
 * Arithmetic follows the reference expression by expression with no FMA
 * contraction (compile with -ffp-contract=off; numba emits none either), and
 * log/sin/cos are the host glibc functions the numba code resolves to, so the
 * oracle is bit-exact with the reference.  That is pinned by
 * tests/test_oracle_golden.py against fingerprints produced by running the
 * reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#ifdef ORACLE_TRACE
#include <stdio.h>
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define LCG_MULT 2806196910506780709ULL
#define LCG_MASK ((1ULL << 63) - 1)
#define STRIDE 152917ULL
#define INV_2_63 (1.0 / 9223372036854775808.0)
#define BELOW_ONE (1.0 - 1.0 / 9007199254740992.0)
#define TWO_PI (2.0 * 3.141592653589793)
#define DIST_EPS 1e-10
#define NUDGE 1e-9
#define MAX_HIST_LOG 100000

enum { SURF_CYL = 0, SURF_XMIN, SURF_XMAX, SURF_YMIN, SURF_YMAX, SURF_ZMIN, SURF_ZMAX, SURF_AXIAL_BASE,
       SURF_LATTICE = 30000 /* extension: internal lattice cell plane */ };
enum { KIND_FUEL = 0, KIND_MOD = 1 };
enum { ROUTE_ERROR = -1, ROUTE_COLLISION = 0, ROUTE_LOOKUP = 1, ROUTE_LEAK = 2, OUT_SCATTER = 0, OUT_DIED = 1 };
enum { CNT_LOG_N = 0, CNT_SITE_N, CNT_OVF, CNT_ERR, CNT_ERR_AUX, CNT_CAPTURES, CNT_FISSIONS,
       CNT_SOURCED, CNT_MAX_DRAWS, CNT_CLAMPS, CNT_INTERP_TRANSPORT, CNT_INTERP_SCORE,
       CNT_EV_LOOKUP, CNT_EV_ADVANCE, CNT_EV_COLLISION, CNT_INV_LOOKUP, CNT_INV_ADVANCE,
       CNT_INV_COLLISION, CNT_SORTS, CNT_MAX_INFLIGHT, CNT_MAX_HIST_LOG, CNT_NUCLIDE_LOOKUPS,
       CNT_LEAKS, CNT_BOX_GUARD };
enum { ERR_NO_SURFACE = 1, ERR_OUTSIDE_BOX, ERR_STREAM_OVERLAP, ERR_RUNAWAY_HISTORY,
       ERR_QUEUE_STATE, ERR_NONPOSITIVE_SIGMA };
enum { TM_LOOKUP = 0, TM_ADVANCE, TM_COLLISION, TM_SORT };

/* Layout mirrors of K:188-190 (lib tuple), K:388-390 (geom), K:567-570 (slots),
 * R:98-105 (log/site buffers).  All pointers are caller-owned numpy memory. */
typedef struct {
    const int64_t *grid_off; const double *grids, *ch_t, *ch_s, *ch_c, *ch_f, *nu;
    const int64_t *mat_off; const int32_t *mat_nuc; const double *mat_den;
    double emin, emax;
} OLib;

typedef struct {
    double radius, r2, hp, height; int64_t n_axial;
    const double *zplanes; const int32_t *fuel_mats; int64_t mod_mat;
    /* extensions (not in the reference): slab layers, vacuum
     * boundaries, track-length mesh (mesh == NULL: off) */
    int32_t slab, vacuum;
    double *mesh; int32_t mnx, mny, mnz, mpad;
    double mx0, my0, mz0, mdx, mdy, mdz;
    /* lattice extension: lat_n x lat_n pin cells of pitch */
    int32_t lat_n, n_pins; double pitch; const int32_t *pin_map; const double *pin_xy;
    /* box guard (extension, RunConfig.box_guard; include/emc.h): 0 = the reference */
    int32_t guard, gpad;
} OGeom;

typedef struct {
    double *px, *py, *pz, *dx, *dy, *dz, *en, *wt;
    uint64_t *rng; int64_t *draws, *gid; int32_t *ordctr, *histlog;
    int8_t *kind; int32_t *axial, *mat;
    double *cm_t, *cm_s, *cm_c, *cm_f, *cm_nsf, *part_t;
    int64_t nslots, part_cols;
} OSlots;

typedef struct {
    int64_t *gid; int32_t *ord, *bin; double *val; int64_t cap;
} OLog;

typedef struct {
    int64_t *parent; int32_t *ord; double *x, *y, *z, *dx, *dy, *dz, *E; int64_t cap;
} OSites;

typedef struct {
    const double *x, *y, *z, *dx, *dy, *dz, *E;
} OSrc;

typedef struct {
    uint64_t seed; int64_t batch, pmax; double alpha, fission_t, k_run;
    int32_t fused, score, use_logs, sort_enabled, sort_every, batch0, history;
    int64_t perturb_gid;
    int32_t fixed_source, pad; double src_energy;     /* extension: fixed surface source */
} OParams;

static double now_s(void) {
    struct timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + (double)ts.tv_nsec * 1e-9;
}

/* K:139-158 */
static inline uint64_t lcg_next(uint64_t s) { return (LCG_MULT * s + 1ULL) & LCG_MASK; }
uint64_t oracle_lcg_skip(uint64_t state, uint64_t n) {
    uint64_t am = 1, aa = 0, cm = LCG_MULT, ca = 1;
    n &= LCG_MASK;
    while (n) {
        if (n & 1) { am = (am * cm) & LCG_MASK; aa = (aa * cm + ca) & LCG_MASK; }
        ca = (ca * (cm + 1)) & LCG_MASK; cm = (cm * cm) & LCG_MASK; n >>= 1;
    }
    return (am * state + aa) & LCG_MASK;
}
/* K:161-169 */
static inline double draw(const OSlots *S, int64_t i) {
    uint64_t s = lcg_next(S->rng[i]);
    S->rng[i] = s; S->draws[i] += 1;
    double u = (double)s * INV_2_63;
    return u >= 1.0 ? BELOW_ONE : u;
}

/* K:393-400 */
static inline int64_t axial_index(double z, int64_t n_axial, double height) {
    int64_t a = (int64_t)((z * (double)n_axial) / height);
    if (a < 0) a = 0; else if (a > n_axial - 1) a = n_axial - 1;
    return a;
}
/* lattice extension: cell of a point, its centre and planes (same
 * operation order as csrc/emc_device.cuh lattice_cell / lattice_lo / _hi) */
static void lattice_cell(const OGeom *g, double x, double y, int32_t *i, int32_t *j, double *cx, double *cy) {
    int32_t a = (int32_t)floor((x + g->hp) / g->pitch), b = (int32_t)floor((y + g->hp) / g->pitch);
    a = a < 0 ? 0 : (a > g->lat_n - 1 ? g->lat_n - 1 : a);
    b = b < 0 ? 0 : (b > g->lat_n - 1 ? g->lat_n - 1 : b);
    *i = a; *j = b;
    *cx = -g->hp + ((double)a + 0.5) * g->pitch;
    *cy = -g->hp + ((double)b + 0.5) * g->pitch;
}
static double lattice_lo(const OGeom *g, int32_t i) { return i == 0 ? -g->hp : -g->hp + (double)i * g->pitch; }
static double lattice_hi(const OGeom *g, int32_t i) {
    return i == g->lat_n - 1 ? g->hp : -g->hp + (double)(i + 1) * g->pitch;
}

/* K:403-415 */
void oracle_locate(double x, double y, double z, const OGeom *g, int64_t *out3) {
    if (x < -g->hp || x > g->hp || y < -g->hp || y > g->hp || z < 0.0 || z > g->height) {
        out3[0] = out3[1] = out3[2] = -1; return;
    }
    if (g->lat_n > 1) {
        int32_t i, j; double cx, cy;
        lattice_cell(g, x, y, &i, &j, &cx, &cy);
        double xl = x - cx, yl = y - cy;
        if (g->pin_map[j * g->lat_n + i] && xl * xl + yl * yl < g->r2) {
            int64_t a = axial_index(z, g->n_axial, g->height);
            out3[0] = KIND_FUEL; out3[1] = a; out3[2] = g->fuel_mats[a]; return;
        }
        out3[0] = KIND_MOD; out3[1] = -1; out3[2] = g->mod_mat; return;
    }
    if (g->slab || x * x + y * y < g->r2) {
        int64_t a = axial_index(z, g->n_axial, g->height);
        out3[0] = KIND_FUEL; out3[1] = a; out3[2] = g->fuel_mats[a]; return;
    }
    out3[0] = KIND_MOD; out3[1] = -1; out3[2] = g->mod_mat;
}
/* K:418-492 */
double oracle_boundary_distance(double x, double y, double z, double ux, double uy, double uz,
                                int64_t kd, int64_t ax, const OGeom *g, int64_t *surf_out) {
    double best = INFINITY, t; int64_t surf = -1;
    double a = ux * ux + uy * uy;
    if (g->lat_n > 1) {          /* lattice extension */
        int32_t li, lj; double cx, cy;
        lattice_cell(g, x, y, &li, &lj, &cx, &cy);
        double xl = x - cx, yl = y - cy;
        int pin = g->pin_map[lj * g->lat_n + li] != 0;
        if (kd == KIND_FUEL) {
            if (a > 0.0) {
                double b = 2.0 * (xl * ux + yl * uy), c = xl * xl + yl * yl - g->r2;
                double disc = b * b - 4.0 * a * c;
                if (disc > 0.0) { t = (-b + sqrt(disc)) / (2.0 * a); if (t > DIST_EPS && t < best) { best = t; surf = SURF_CYL; } }
            }
            if (uz > 0.0) {
                t = (g->zplanes[ax + 1] - z) / uz;
                if (t > DIST_EPS && t < best) { best = t; surf = ax == g->n_axial - 1 ? SURF_ZMAX : SURF_AXIAL_BASE + ax + 1; }
            } else if (uz < 0.0) {
                t = (g->zplanes[ax] - z) / uz;
                if (t > DIST_EPS && t < best) { best = t; surf = ax == 0 ? SURF_ZMIN : SURF_AXIAL_BASE + ax; }
            }
        } else {
            if (pin && a > 0.0) {
                double b = 2.0 * (xl * ux + yl * uy), c = xl * xl + yl * yl - g->r2;
                double disc = b * b - 4.0 * a * c;
                if (disc > 0.0) { t = (-b - sqrt(disc)) / (2.0 * a); if (t > DIST_EPS && t < best) { best = t; surf = SURF_CYL; } }
            }
            if (ux > 0.0) { t = (lattice_hi(g, li) - x) / ux; if (t > DIST_EPS && t < best) { best = t; surf = li == g->lat_n - 1 ? SURF_XMAX : SURF_LATTICE; } }
            else if (ux < 0.0) { t = (lattice_lo(g, li) - x) / ux; if (t > DIST_EPS && t < best) { best = t; surf = li == 0 ? SURF_XMIN : SURF_LATTICE; } }
            if (uy > 0.0) { t = (lattice_hi(g, lj) - y) / uy; if (t > DIST_EPS && t < best) { best = t; surf = lj == g->lat_n - 1 ? SURF_YMAX : SURF_LATTICE; } }
            else if (uy < 0.0) { t = (lattice_lo(g, lj) - y) / uy; if (t > DIST_EPS && t < best) { best = t; surf = lj == 0 ? SURF_YMIN : SURF_LATTICE; } }
            if (uz > 0.0) { t = (g->height - z) / uz; if (t > DIST_EPS && t < best) { best = t; surf = SURF_ZMAX; } }
            else if (uz < 0.0) { t = (0.0 - z) / uz; if (t > DIST_EPS && t < best) { best = t; surf = SURF_ZMIN; } }
        }
        *surf_out = surf;
        return best;
    }
    if (kd == KIND_FUEL) {
        if (g->slab) {    /* extension: slab layer bounded by the box side planes */
            if (ux > 0.0) { t = (g->hp - x) / ux; if (t > DIST_EPS && t < best) { best = t; surf = SURF_XMAX; } }
            else if (ux < 0.0) { t = (-g->hp - x) / ux; if (t > DIST_EPS && t < best) { best = t; surf = SURF_XMIN; } }
            if (uy > 0.0) { t = (g->hp - y) / uy; if (t > DIST_EPS && t < best) { best = t; surf = SURF_YMAX; } }
            else if (uy < 0.0) { t = (-g->hp - y) / uy; if (t > DIST_EPS && t < best) { best = t; surf = SURF_YMIN; } }
        } else if (a > 0.0) {
            double b = 2.0 * (x * ux + y * uy), c = x * x + y * y - g->r2;
            double disc = b * b - 4.0 * a * c;
            if (disc > 0.0) { t = (-b + sqrt(disc)) / (2.0 * a); if (t > DIST_EPS && t < best) { best = t; surf = SURF_CYL; } }
        }
        if (uz > 0.0) {
            t = (g->zplanes[ax + 1] - z) / uz;
            if (t > DIST_EPS && t < best) { best = t; surf = ax == g->n_axial - 1 ? SURF_ZMAX : SURF_AXIAL_BASE + ax + 1; }
        } else if (uz < 0.0) {
            t = (g->zplanes[ax] - z) / uz;
            if (t > DIST_EPS && t < best) { best = t; surf = ax == 0 ? SURF_ZMIN : SURF_AXIAL_BASE + ax; }
        }
    } else {
        if (a > 0.0) {
            double b = 2.0 * (x * ux + y * uy), c = x * x + y * y - g->r2;
            double disc = b * b - 4.0 * a * c;
            if (disc > 0.0) { t = (-b - sqrt(disc)) / (2.0 * a); if (t > DIST_EPS && t < best) { best = t; surf = SURF_CYL; } }
        }
        if (ux > 0.0) { t = (g->hp - x) / ux; if (t > DIST_EPS && t < best) { best = t; surf = SURF_XMAX; } }
        else if (ux < 0.0) { t = (-g->hp - x) / ux; if (t > DIST_EPS && t < best) { best = t; surf = SURF_XMIN; } }
        if (uy > 0.0) { t = (g->hp - y) / uy; if (t > DIST_EPS && t < best) { best = t; surf = SURF_YMAX; } }
        else if (uy < 0.0) { t = (-g->hp - y) / uy; if (t > DIST_EPS && t < best) { best = t; surf = SURF_YMIN; } }
        if (uz > 0.0) { t = (g->height - z) / uz; if (t > DIST_EPS && t < best) { best = t; surf = SURF_ZMAX; } }
        else if (uz < 0.0) { t = (0.0 - z) / uz; if (t > DIST_EPS && t < best) { best = t; surf = SURF_ZMIN; } }
    }
    *surf_out = surf;
    return best;
}
/* K:495-501 */
void oracle_isotropic(double u1, double u2, double *out3) {
    double mu = 2.0 * u1 - 1.0, phi = TWO_PI * u2, s = sqrt(1.0 - mu * mu);
    out3[0] = s * cos(phi); out3[1] = s * sin(phi); out3[2] = mu;
}

/* per-nuclide bracket search, K:614-621 (binary search, "last grid <= E") */
static inline int64_t bracket(const double *grids, int64_t g0, int64_t g1, double E) {
    int64_t ii = g0, bb = g1 - 1;
    while (bb - ii > 1) { int64_t mid = (ii + bb) >> 1; if (grids[mid] <= E) ii = mid; else bb = mid; }
    return ii;
}

/* K:287-331 (binary backend; the three backends are bit-identical by K:1-23) */
void oracle_macro_lookup(const OLib *L, int64_t m, double E, double *sums5, double *part_out) {
    int64_t e0 = L->mat_off[m], e1 = L->mat_off[m + 1];
    double st = 0.0, ss = 0.0, sc = 0.0, sf = 0.0, snf = 0.0;
    for (int64_t k = e0; k < e1; ++k) {
        int32_t nid = L->mat_nuc[k]; double den = L->mat_den[k];
        int64_t g0 = L->grid_off[nid], g1 = L->grid_off[nid + 1];
        double t, s, c, f;
        if (E <= L->grids[g0]) { t = L->ch_t[g0]; s = L->ch_s[g0]; c = L->ch_c[g0]; f = L->ch_f[g0]; }
        else if (E >= L->grids[g1 - 1]) { int64_t p = g1 - 1; t = L->ch_t[p]; s = L->ch_s[p]; c = L->ch_c[p]; f = L->ch_f[p]; }
        else {
            int64_t i = bracket(L->grids, g0, g1, E);
            double fr = (E - L->grids[i]) / (L->grids[i + 1] - L->grids[i]);
            t = L->ch_t[i] + fr * (L->ch_t[i + 1] - L->ch_t[i]);
            s = L->ch_s[i] + fr * (L->ch_s[i + 1] - L->ch_s[i]);
            c = L->ch_c[i] + fr * (L->ch_c[i + 1] - L->ch_c[i]);
            f = L->ch_f[i] + fr * (L->ch_f[i + 1] - L->ch_f[i]);
        }
        double pt = den * t;
        st += pt; ss += den * s; sc += den * c; sf += den * f; snf += den * L->nu[nid] * f;
        if (part_out) {
            double *p = part_out + 4 * (k - e0);
            p[0] = pt; p[1] = den * s; p[2] = den * c; p[3] = den * f;
        }
    }
    sums5[0] = st; sums5[1] = ss; sums5[2] = sc; sums5[3] = sf; sums5[4] = snf;
}

/* K:509-530 */
static int log_append(OLog *lg, int64_t *cnt, int64_t g, const OSlots *S, int64_t i, int32_t bin, double val) {
    if (val == 0.0) return 0;
    int64_t n = cnt[CNT_LOG_N];
    if (n >= lg->cap) { cnt[CNT_OVF] = 1; return -1; }
    lg->gid[n] = g; lg->ord[n] = S->ordctr[i]; lg->bin[n] = bin; lg->val[n] = val;
    cnt[CNT_LOG_N] = n + 1;
    S->ordctr[i] += 1; S->histlog[i] += 1;
    if (S->histlog[i] > MAX_HIST_LOG) { cnt[CNT_ERR] = ERR_RUNAWAY_HISTORY; cnt[CNT_ERR_AUX] = g; return -1; }
    return 0;
}
/* K:533-550 */
static int site_append(OSites *sb, int64_t *cnt, int64_t parent, int32_t ord, double x, double y, double z,
                       double ux, double uy, double uz, double E) {
    int64_t n = cnt[CNT_SITE_N];
    if (n >= sb->cap) { cnt[CNT_OVF] = 2; return -1; }
    sb->parent[n] = parent; sb->ord[n] = ord; sb->x[n] = x; sb->y[n] = y; sb->z[n] = z;
    sb->dx[n] = ux; sb->dy[n] = uy; sb->dz[n] = uz; sb->E[n] = E;
    cnt[CNT_SITE_N] = n + 1;
    return 0;
}
/* K:553-561 */
static inline double clamp_energy(double E, const OLib *L, int64_t *cnt) {
    if (E < L->emin) { cnt[CNT_CLAMPS] += 1; return L->emin; }
    if (E > L->emax) { cnt[CNT_CLAMPS] += 1; return L->emax; }
    return E;
}

/* K:573-710 (fused keeps part_t) */
static void op_lookup(int64_t i, const OSlots *S, const OLib *L, int fused, int64_t *cnt) {
    double E = S->en[i]; int64_t m = S->mat[i];
    int64_t e0 = L->mat_off[m], e1 = L->mat_off[m + 1];
    double st = 0.0, ss = 0.0, sc = 0.0, sf = 0.0, snf = 0.0;
    for (int64_t k = e0; k < e1; ++k) {
        int32_t nid = L->mat_nuc[k]; double den = L->mat_den[k];
        int64_t g0 = L->grid_off[nid], g1 = L->grid_off[nid + 1];
        double t, s, c, f;
        if (E <= L->grids[g0]) { t = L->ch_t[g0]; s = L->ch_s[g0]; c = L->ch_c[g0]; f = L->ch_f[g0]; }
        else if (E >= L->grids[g1 - 1]) { int64_t p = g1 - 1; t = L->ch_t[p]; s = L->ch_s[p]; c = L->ch_c[p]; f = L->ch_f[p]; }
        else {
            int64_t ii = bracket(L->grids, g0, g1, E);
            double fr = (E - L->grids[ii]) / (L->grids[ii + 1] - L->grids[ii]);
            t = L->ch_t[ii] + fr * (L->ch_t[ii + 1] - L->ch_t[ii]);
            s = L->ch_s[ii] + fr * (L->ch_s[ii + 1] - L->ch_s[ii]);
            c = L->ch_c[ii] + fr * (L->ch_c[ii + 1] - L->ch_c[ii]);
            f = L->ch_f[ii] + fr * (L->ch_f[ii + 1] - L->ch_f[ii]);
        }
        double pt = den * t;
        st += pt; ss += den * s; sc += den * c; sf += den * f; snf += den * L->nu[nid] * f;
        if (fused) S->part_t[i * S->part_cols + (k - e0)] = pt;
    }
    S->cm_t[i] = st; S->cm_s[i] = ss; S->cm_c[i] = sc; S->cm_f[i] = sf; S->cm_nsf[i] = snf;
    cnt[CNT_INTERP_TRANSPORT] += 4 * (e1 - e0);
}

/* K:334-382 naive scoring re-loop */
static void reassemble_tcf(double E, int64_t m, const OLib *L, double *o4) {
    int64_t e0 = L->mat_off[m], e1 = L->mat_off[m + 1];
    double st = 0.0, sc = 0.0, sf = 0.0, snf = 0.0;
    for (int64_t k = e0; k < e1; ++k) {
        int32_t nid = L->mat_nuc[k]; double den = L->mat_den[k];
        int64_t g0 = L->grid_off[nid], g1 = L->grid_off[nid + 1];
        double t, c, f;
        if (E <= L->grids[g0]) { t = L->ch_t[g0]; c = L->ch_c[g0]; f = L->ch_f[g0]; }
        else if (E >= L->grids[g1 - 1]) { int64_t p = g1 - 1; t = L->ch_t[p]; c = L->ch_c[p]; f = L->ch_f[p]; }
        else {
            int64_t i = bracket(L->grids, g0, g1, E);
            double fr = (E - L->grids[i]) / (L->grids[i + 1] - L->grids[i]);
            t = L->ch_t[i] + fr * (L->ch_t[i + 1] - L->ch_t[i]);
            c = L->ch_c[i] + fr * (L->ch_c[i + 1] - L->ch_c[i]);
            f = L->ch_f[i] + fr * (L->ch_f[i + 1] - L->ch_f[i]);
        }
        st += den * t; sc += den * c; sf += den * f; snf += den * L->nu[nid] * f;
    }
    o4[0] = st; o4[1] = sc; o4[2] = sf; o4[3] = snf;
}

/* Extension: track-length mesh estimator, the same 3D DDA
 * and operation order as the device (csrc/emc_device.cuh: score_mesh). */
static inline int32_t mesh_cell(double v, double v0, double dv, int32_t n) {
    int32_t i = (int32_t)floor((v - v0) / dv);
    return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
}
static inline double mesh_next(double v, double u, int32_t i, double v0, double dv) {
    if (u > 0.0) return ((v0 + (double)(i + 1) * dv) - v) / u;
    if (u < 0.0) return ((v0 + (double)i * dv) - v) / u;
    return INFINITY;
}
static void mesh_score(const OGeom *G, double x, double y, double z, double ux, double uy, double uz,
                       double ell, double sig_t) {
    int32_t ix = mesh_cell(x, G->mx0, G->mdx, G->mnx), iy = mesh_cell(y, G->my0, G->mdy, G->mny),
            iz = mesh_cell(z, G->mz0, G->mdz, G->mnz);
    double t = 0.0;
    for (;;) {
        double tx = mesh_next(x, ux, ix, G->mx0, G->mdx), ty = mesh_next(y, uy, iy, G->my0, G->mdy),
               tz = mesh_next(z, uz, iz, G->mz0, G->mdz);
        double tn = tx < ty ? tx : ty;
        tn = tz < tn ? tz : tn;
        int last = !(tn < ell);
        if (last) tn = ell;
        double seg = tn - t;
        if (seg > 0.0) {
            double *a = G->mesh + 2 * (((int64_t)iz * G->mny + iy) * G->mnx + ix);
            a[0] += seg; a[1] += seg * sig_t;
        }
        if (last) break;
        if (tx == tn) { ix += ux > 0.0 ? 1 : -1; if (ix < 0 || ix >= G->mnx) break; }
        else if (ty == tn) { iy += uy > 0.0 ? 1 : -1; if (iy < 0 || iy >= G->mny) break; }
        else { iz += uz > 0.0 ? 1 : -1; if (iz < 0 || iz >= G->mnz) break; }
        if (tn > t) t = tn;
    }
}

/* Box guard (extension, off by default; include/emc.h): the reference can
 * leave a particle outside the reflective box -- e.g. an axial-plane crossing
 * within 1e-9 of the cylinder nudges a fuel particle out of the cylinder while
 * its cell stays fuel, and fuel cells never test the box planes (K:430-450,
 * K:796-811).  A particle outside the closed box after a move is put back on
 * the face it passed with that direction component pointing inward. */
static int guard_fold(double *x, double *y, double *z, double *dx, double *dy, double *dz, const OGeom *G) {
    int out = 0;
    if (*x > G->hp) { *x = G->hp; if (*dx > 0.0) *dx = -*dx; out = 1; }
    else if (*x < -G->hp) { *x = -G->hp; if (*dx < 0.0) *dx = -*dx; out = 1; }
    if (*y > G->hp) { *y = G->hp; if (*dy > 0.0) *dy = -*dy; out = 1; }
    else if (*y < -G->hp) { *y = -G->hp; if (*dy < 0.0) *dy = -*dy; out = 1; }
    if (*z > G->height) { *z = G->height; if (*dz > 0.0) *dz = -*dz; out = 1; }
    else if (*z < 0.0) { *z = 0.0; if (*dz < 0.0) *dz = -*dz; out = 1; }
    return out;
}
/* ... then its cell is re-located and it goes back to the lookup queue (no
 * collision at the guarded point); with vacuum planes it leaks. */
static int guard_route(int64_t i, const OSlots *S, const OGeom *G, int64_t *cnt) {
    cnt[CNT_BOX_GUARD] += 1;
    if (G->vacuum) { cnt[CNT_LEAKS] += 1; return ROUTE_LEAK; }
    int64_t loc[3];
    oracle_locate(S->px[i], S->py[i], S->pz[i], G, loc);
    S->kind[i] = (int8_t)loc[0]; S->axial[i] = (int32_t)loc[1]; S->mat[i] = (int32_t)loc[2];
    return ROUTE_LOOKUP;
}
#define GUARD(i) (G->guard && guard_fold(&S->px[i], &S->py[i], &S->pz[i], &S->dx[i], &S->dy[i], &S->dz[i], G))

/* K:713-811 */
static int op_advance(int64_t i, const OSlots *S, const OLib *L, const OGeom *G, OLog *lg, double *wbins,
                      int64_t *cnt, int score, int fused, int use_logs) {
    double sig_t = S->cm_t[i];
    if (sig_t <= 0.0) { cnt[CNT_ERR] = ERR_NONPOSITIVE_SIGMA; cnt[CNT_ERR_AUX] = S->gid[i]; return ROUTE_ERROR; }
    double u = draw(S, i);
    double d_coll = -log(1.0 - u) / sig_t;
    int64_t surf;
    double dist = oracle_boundary_distance(S->px[i], S->py[i], S->pz[i], S->dx[i], S->dy[i], S->dz[i],
                                           S->kind[i], S->axial[i], G, &surf);
    if (surf < 0) { cnt[CNT_ERR] = ERR_NO_SURFACE; cnt[CNT_ERR_AUX] = S->gid[i]; return ROUTE_ERROR; }
    double ell; int crossing;
    if (d_coll < dist) { ell = d_coll; crossing = 0; } else { ell = dist; crossing = 1; }
    if (score) {
        int64_t region = S->kind[i] == KIND_FUEL ? (int64_t)S->axial[i] : G->n_axial;
        int32_t base = (int32_t)(region * 5);
        double fl = S->wt[i] * ell, v_tot, v_abs, v_fis, v_nsf;
        if (fused) {
            v_tot = fl * sig_t; v_abs = fl * (S->cm_c[i] + S->cm_f[i]); v_fis = fl * S->cm_f[i]; v_nsf = fl * S->cm_nsf[i];
        } else {
            double o4[4]; int64_t m = S->mat[i];
            reassemble_tcf(S->en[i], m, L, o4);
            cnt[CNT_INTERP_SCORE] += 3 * (L->mat_off[m + 1] - L->mat_off[m]);
            v_tot = fl * o4[0]; v_abs = fl * (o4[1] + o4[2]); v_fis = fl * o4[2]; v_nsf = fl * o4[3];
        }
        if (use_logs) {
            int64_t g = S->gid[i];
            log_append(lg, cnt, g, S, i, base + 0, fl);
            log_append(lg, cnt, g, S, i, base + 1, v_tot);
            log_append(lg, cnt, g, S, i, base + 2, v_abs);
            log_append(lg, cnt, g, S, i, base + 3, v_fis);
            log_append(lg, cnt, g, S, i, base + 4, v_nsf);
            if (cnt[CNT_OVF] != 0 || cnt[CNT_ERR] != 0) return ROUTE_ERROR;
        } else {
            wbins[base + 0] += fl; wbins[base + 1] += v_tot; wbins[base + 2] += v_abs;
            wbins[base + 3] += v_fis; wbins[base + 4] += v_nsf;
        }
        if (G->mesh) mesh_score(G, S->px[i], S->py[i], S->pz[i], S->dx[i], S->dy[i], S->dz[i], ell, sig_t);
    }
#ifdef ORACLE_TRACE   /* tools/c4_escape_replay.py --trace: one line per advance */
    fprintf(stderr, "adv gid=%lld kind=%d ax=%d pos=(%.17g,%.17g,%.17g) dir=(%.17g,%.17g,%.17g) E=%.17g "
            "d_coll=%.17g dist=%.17g surf=%lld\n", (long long)S->gid[i], S->kind[i], S->axial[i], S->px[i],
            S->py[i], S->pz[i], S->dx[i], S->dy[i], S->dz[i], S->en[i], d_coll, dist, (long long)surf);
#endif
    S->px[i] += S->dx[i] * ell; S->py[i] += S->dy[i] * ell; S->pz[i] += S->dz[i] * ell;
    if (!crossing) return GUARD(i) ? guard_route(i, S, G, cnt) : ROUTE_COLLISION;
    if (G->vacuum && surf >= SURF_XMIN && surf <= SURF_ZMAX) { cnt[CNT_LEAKS] += 1; return ROUTE_LEAK; }
    if (surf >= SURF_XMIN && surf <= SURF_ZMAX) {
        if (surf == SURF_XMIN || surf == SURF_XMAX) S->dx[i] = -S->dx[i];
        else if (surf == SURF_YMIN || surf == SURF_YMAX) S->dy[i] = -S->dy[i];
        else S->dz[i] = -S->dz[i];
    }
    S->px[i] += S->dx[i] * NUDGE; S->py[i] += S->dy[i] * NUDGE; S->pz[i] += S->dz[i] * NUDGE;
    if (surf == SURF_CYL) {
        if (S->kind[i] == KIND_FUEL) { S->kind[i] = KIND_MOD; S->axial[i] = -1; }
        else { S->kind[i] = KIND_FUEL; S->axial[i] = (int32_t)axial_index(S->pz[i], G->n_axial, G->height); }
    } else if (surf >= SURF_AXIAL_BASE && surf < SURF_LATTICE) {
        int64_t jpl = surf - SURF_AXIAL_BASE;
        S->axial[i] = (int32_t)(S->dz[i] > 0.0 ? jpl : jpl - 1);
    }
    S->mat[i] = S->kind[i] == KIND_FUEL ? G->fuel_mats[S->axial[i]] : (int32_t)G->mod_mat;
    return GUARD(i) ? guard_route(i, S, G, cnt) : ROUTE_LOOKUP;
}

/* K:814-923 */
static int op_collision(int64_t i, const OSlots *S, const OLib *L, OLog *lg, OSites *sb, double *wbins,
                        int64_t *cnt, const OParams *P, int32_t kbin) {
    double st = S->cm_t[i]; int64_t g = S->gid[i];
    double kval = S->wt[i] * (S->cm_nsf[i] / st);
    if (P->use_logs) { if (log_append(lg, cnt, g, S, i, kbin, kval) < 0) return ROUTE_ERROR; }
    else wbins[kbin] += kval;
    double E = S->en[i]; int64_t m = S->mat[i];
    int64_t e0 = L->mat_off[m], e1 = L->mat_off[m + 1];
    double u1 = draw(S, i), tgt = u1 * st, cum = 0.0, pt_sel = 0.0;
    int64_t ksel = e1 - 1;
    if (P->fused) {
        for (int64_t k = e0; k < e1; ++k) {
            double pt = S->part_t[i * S->part_cols + (k - e0)];
            pt_sel = pt;
            if (cum + pt > tgt) { ksel = k; break; }
            cum += pt;
        }
    } else {
        for (int64_t k = e0; k < e1; ++k) {
            int32_t nid = L->mat_nuc[k];
            int64_t g0 = L->grid_off[nid], g1 = L->grid_off[nid + 1];
            double t;
            if (E <= L->grids[g0]) t = L->ch_t[g0];
            else if (E >= L->grids[g1 - 1]) t = L->ch_t[g1 - 1];
            else {
                int64_t ii = bracket(L->grids, g0, g1, E);
                double fr = (E - L->grids[ii]) / (L->grids[ii + 1] - L->grids[ii]);
                t = L->ch_t[ii] + fr * (L->ch_t[ii + 1] - L->ch_t[ii]);
            }
            double pt = L->mat_den[k] * t;
            cnt[CNT_INTERP_TRANSPORT] += 1;
            pt_sel = pt;
            if (cum + pt > tgt) { ksel = k; break; }
            cum += pt;
        }
    }
    int32_t nid_sel = L->mat_nuc[ksel]; double den_sel = L->mat_den[ksel];
    int64_t g0 = L->grid_off[nid_sel], g1 = L->grid_off[nid_sel + 1];
    double s_s, s_c, s_f;     /* K:257-274 */
    if (E <= L->grids[g0]) { s_s = L->ch_s[g0]; s_c = L->ch_c[g0]; s_f = L->ch_f[g0]; }
    else if (E >= L->grids[g1 - 1]) { int64_t p = g1 - 1; s_s = L->ch_s[p]; s_c = L->ch_c[p]; s_f = L->ch_f[p]; }
    else {
        int64_t ii = bracket(L->grids, g0, g1, E);
        double fr = (E - L->grids[ii]) / (L->grids[ii + 1] - L->grids[ii]);
        s_s = L->ch_s[ii] + fr * (L->ch_s[ii + 1] - L->ch_s[ii]);
        s_c = L->ch_c[ii] + fr * (L->ch_c[ii + 1] - L->ch_c[ii]);
        s_f = L->ch_f[ii] + fr * (L->ch_f[ii + 1] - L->ch_f[ii]);
    }
    (void)s_f;
    cnt[CNT_INTERP_TRANSPORT] += 3;
    double ps = den_sel * s_s, pc = den_sel * s_c;
    double u2 = draw(S, i), tgt2 = u2 * pt_sel;
    if (tgt2 < ps) {
        double u3 = draw(S, i), u4 = draw(S, i), d3[3];
        oracle_isotropic(u3, u4, d3);
        S->dx[i] = d3[0]; S->dy[i] = d3[1]; S->dz[i] = d3[2];
        double u5 = draw(S, i);
        double ep = E * (P->alpha + (1.0 - P->alpha) * u5);
        S->en[i] = clamp_energy(ep, L, cnt);
        return OUT_SCATTER;
    }
    if (tgt2 < ps + pc) { cnt[CNT_CAPTURES] += 1; return OUT_DIED; }
    cnt[CNT_FISSIONS] += 1;
    double nu_sel = L->nu[nid_sel];
    double u5 = draw(S, i);
    int64_t nsites = (int64_t)floor(nu_sel / P->k_run + u5);
    for (int64_t ms = 0; ms < nsites; ++ms) {
        double ua = draw(S, i), ub = draw(S, i), d3[3];
        oracle_isotropic(ua, ub, d3);
        double uc = draw(S, i);
        double es = clamp_energy(-P->fission_t * log(1.0 - uc), L, cnt);
        if (site_append(sb, cnt, g, (int32_t)ms, S->px[i], S->py[i], S->pz[i], d3[0], d3[1], d3[2], es) < 0)
            return ROUTE_ERROR;
    }
    return OUT_DIED;
}

/* K:926-996 */
static int op_source(int64_t i, int64_t g, const OSlots *S, const OLib *L, const OGeom *G, const OSrc *src,
                     const OParams *P, int64_t *cnt) {
    uint64_t offset = ((uint64_t)P->batch * (uint64_t)P->pmax + (uint64_t)g) * STRIDE;
    uint64_t s0 = oracle_lcg_skip(P->seed, offset);
    if (g == P->perturb_gid) s0 ^= 1ULL;
    S->rng[i] = s0; S->draws[i] = 0; S->ordctr[i] = 0; S->histlog[i] = 0; S->gid[i] = g; S->wt[i] = 1.0;
    if (P->fixed_source) {    /* extension: surface source on z = 0, mu = u inward */
        double u1 = draw(S, i), u2 = draw(S, i);
        S->px[i] = (2.0 * u1 - 1.0) * G->hp; S->py[i] = (2.0 * u2 - 1.0) * G->hp; S->pz[i] = 0.0;
        double mu = draw(S, i), phi = TWO_PI * draw(S, i), sn = sqrt(1.0 - mu * mu);
        S->dx[i] = sn * cos(phi); S->dy[i] = sn * sin(phi); S->dz[i] = mu;
        if (P->src_energy > 0.0) S->en[i] = P->src_energy;
        else { double ue = draw(S, i); S->en[i] = clamp_energy(-P->fission_t * log(1.0 - ue), L, cnt); }
    } else if (P->batch0) {
        double x, y, cx = 0.0, cy = 0.0;
        if (G->lat_n > 1) {    /* lattice extension: uniform fuel pin, then its disk */
            int64_t k = (int64_t)(draw(S, i) * (double)G->n_pins);
            if (k > G->n_pins - 1) k = G->n_pins - 1;
            cx = G->pin_xy[2 * k]; cy = G->pin_xy[2 * k + 1];
        }
        for (;;) {
            double u1 = draw(S, i), u2 = draw(S, i);
            x = (2.0 * u1 - 1.0) * G->radius; y = (2.0 * u2 - 1.0) * G->radius;
            if (x * x + y * y < G->r2) break;
            if (S->draws[i] >= (int64_t)STRIDE) { cnt[CNT_ERR] = ERR_STREAM_OVERLAP; cnt[CNT_ERR_AUX] = g; return -1; }
        }
        if (G->lat_n > 1) { x = cx + x; y = cy + y; }
        double z = draw(S, i) * G->height;
        double ua = draw(S, i), ub = draw(S, i), d3[3];
        oracle_isotropic(ua, ub, d3);
        double ue = draw(S, i);
        double e = clamp_energy(-P->fission_t * log(1.0 - ue), L, cnt);
        S->px[i] = x; S->py[i] = y; S->pz[i] = z; S->dx[i] = d3[0]; S->dy[i] = d3[1]; S->dz[i] = d3[2]; S->en[i] = e;
    } else {
        S->px[i] = src->x[g]; S->py[i] = src->y[g]; S->pz[i] = src->z[g];
        S->dx[i] = src->dx[g]; S->dy[i] = src->dy[g]; S->dz[i] = src->dz[g]; S->en[i] = src->E[g];
    }
    int64_t loc[3];
    oracle_locate(S->px[i], S->py[i], S->pz[i], G, loc);
    if (loc[0] < 0) { cnt[CNT_ERR] = ERR_OUTSIDE_BOX; cnt[CNT_ERR_AUX] = g; return -1; }
    S->kind[i] = (int8_t)loc[0]; S->axial[i] = (int32_t)loc[1]; S->mat[i] = (int32_t)loc[2];
    return 0;
}

/* K:999-1006 */
static void finish_history(int64_t i, const OSlots *S, int64_t *cnt) {
    if (S->draws[i] > cnt[CNT_MAX_DRAWS]) cnt[CNT_MAX_DRAWS] = S->draws[i];
    if (S->histlog[i] > cnt[CNT_MAX_HIST_LOG]) cnt[CNT_MAX_HIST_LOG] = S->histlog[i];
}

/* K:1014-1035: stable sort by (material, energy) == sort by (mat, E, position) */
typedef struct { int32_t mat; double e; int64_t pos; int32_t slot; } OKey;
static int key_cmp(const void *a, const void *b) {
    const OKey *x = a, *y = b;
    if (x->mat != y->mat) return x->mat < y->mat ? -1 : 1;
    if (x->e != y->e) return x->e < y->e ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}
void oracle_sort_queue(int32_t *q, int64_t n, const int32_t *mat, const double *en) {
    OKey *k = malloc(sizeof(OKey) * (n ? n : 1));
    for (int64_t t = 0; t < n; ++t) { k[t].mat = mat[q[t]]; k[t].e = en[q[t]]; k[t].pos = t; k[t].slot = q[t]; }
    qsort(k, (size_t)n, sizeof(OKey), key_cmp);
    for (int64_t t = 0; t < n; ++t) q[t] = k[t].slot;
    free(k);
}

/* K:1043-1089 */
static void run_history_batch(const int64_t *assigned, int64_t n_assigned, const OSlots *S, const OLib *L,
                              const OGeom *G, const OSrc *src, OLog *lg, OSites *sb, double *wbins, int32_t nbins,
                              int64_t *cnt, double *tm, const OParams *P) {
    for (int64_t ai = 0; ai < n_assigned; ++ai) {
        if (op_source(0, assigned[ai], S, L, G, src, P, cnt) < 0) return;
        cnt[CNT_SOURCED] += 1;
        int alive = 1;
        while (alive) {
            double t0 = now_s();
            op_lookup(0, S, L, P->fused, cnt);
            double t1 = now_s(); tm[TM_LOOKUP] += t1 - t0;
            cnt[CNT_EV_LOOKUP] += 1; cnt[CNT_INV_LOOKUP] += 1;
            int r = op_advance(0, S, L, G, lg, wbins, cnt, P->score, P->fused, P->use_logs);
            double t2 = now_s(); tm[TM_ADVANCE] += t2 - t1;
            cnt[CNT_EV_ADVANCE] += 1; cnt[CNT_INV_ADVANCE] += 1;
            if (r == ROUTE_ERROR) return;
            if (r == ROUTE_LEAK) alive = 0;
            if (r == ROUTE_COLLISION) {
                int rc = op_collision(0, S, L, lg, sb, wbins, cnt, P, nbins - 1);
                double t3 = now_s(); tm[TM_COLLISION] += t3 - t2;
                cnt[CNT_EV_COLLISION] += 1; cnt[CNT_INV_COLLISION] += 1;
                if (rc == ROUTE_ERROR) return;
                if (rc == OUT_DIED) alive = 0;
            }
            if (S->draws[0] >= (int64_t)STRIDE) { cnt[CNT_ERR] = ERR_STREAM_OVERLAP; cnt[CNT_ERR_AUX] = S->gid[0]; return; }
        }
        finish_history(0, S, cnt);
    }
    cnt[CNT_MAX_INFLIGHT] = 1;
}

/* K:1092-1211 */
static void run_event_batch(const int64_t *assigned, int64_t n_assigned, const OSlots *S, const OLib *L,
                            const OGeom *G, const OSrc *src, OLog *lg, OSites *sb, double *wbins, int32_t nbins,
                            int64_t *cnt, double *tm, const OParams *P) {
    int64_t nslots = S->nslots;
    int32_t *q_look = malloc(sizeof(int32_t) * nslots), *q_adv = malloc(sizeof(int32_t) * nslots),
            *q_col = malloc(sizeof(int32_t) * nslots);
    int64_t nl = 0, na = 0, nc = 0, cursor = 0, inflight = 0;
    while (cursor < n_assigned && inflight < nslots) {
        if (op_source(inflight, assigned[cursor], S, L, G, src, P, cnt) < 0) goto done;
        q_look[nl++] = (int32_t)inflight; cursor++; inflight++; cnt[CNT_SOURCED] += 1;
    }
    if (inflight > cnt[CNT_MAX_INFLIGHT]) cnt[CNT_MAX_INFLIGHT] = inflight;
    int64_t look_inv = 0;
    int32_t kbin = nbins - 1;
    while (nl + na + nc > 0) {
        if (nl >= na && nl >= nc) {
            if (P->sort_enabled && nl > 1 && look_inv % P->sort_every == 0) {
                double t0 = now_s();
                oracle_sort_queue(q_look, nl, S->mat, S->en);
                tm[TM_SORT] += now_s() - t0; cnt[CNT_SORTS] += 1;
            }
            look_inv++;
            double t0 = now_s();
            for (int64_t qi = 0; qi < nl; ++qi) { int32_t s = q_look[qi]; op_lookup(s, S, L, P->fused, cnt); q_adv[na++] = s; }
            tm[TM_LOOKUP] += now_s() - t0;
            cnt[CNT_EV_LOOKUP] += nl; cnt[CNT_INV_LOOKUP] += 1; nl = 0;
        } else if (na >= nc) {
            double t0 = now_s(); int64_t n_sweep = na;
            for (int64_t qi = 0; qi < n_sweep; ++qi) {
                int32_t s = q_adv[qi];
                int r = op_advance(s, S, L, G, lg, wbins, cnt, P->score, P->fused, P->use_logs);
                if (r == ROUTE_ERROR) goto done;
                if (S->draws[s] >= (int64_t)STRIDE) { cnt[CNT_ERR] = ERR_STREAM_OVERLAP; cnt[CNT_ERR_AUX] = S->gid[s]; goto done; }
                if (r == ROUTE_COLLISION) q_col[nc++] = s;
                else if (r == ROUTE_LEAK) {             /* extension: vacuum leakage ends the history */
                    finish_history(s, S, cnt); inflight--;
                    if (cursor < n_assigned) {
                        if (op_source(s, assigned[cursor], S, L, G, src, P, cnt) < 0) goto done;
                        cursor++; inflight++; cnt[CNT_SOURCED] += 1; q_look[nl++] = s;
                    }
                } else q_look[nl++] = s;
            }
            tm[TM_ADVANCE] += now_s() - t0;
            cnt[CNT_EV_ADVANCE] += n_sweep; cnt[CNT_INV_ADVANCE] += 1; na = 0;
        } else {
            double t0 = now_s(); int64_t n_sweep = nc;
            for (int64_t qi = 0; qi < n_sweep; ++qi) {
                int32_t s = q_col[qi];
                int rc = op_collision(s, S, L, lg, sb, wbins, cnt, P, kbin);
                if (rc == ROUTE_ERROR) goto done;
                if (S->draws[s] >= (int64_t)STRIDE) { cnt[CNT_ERR] = ERR_STREAM_OVERLAP; cnt[CNT_ERR_AUX] = S->gid[s]; goto done; }
                if (rc == OUT_SCATTER) q_look[nl++] = s;
                else {
                    finish_history(s, S, cnt); inflight--;
                    if (cursor < n_assigned) {
                        if (op_source(s, assigned[cursor], S, L, G, src, P, cnt) < 0) goto done;
                        cursor++; inflight++; cnt[CNT_SOURCED] += 1; q_look[nl++] = s;
                    }
                }
            }
            tm[TM_COLLISION] += now_s() - t0;
            cnt[CNT_EV_COLLISION] += n_sweep; cnt[CNT_INV_COLLISION] += 1; nc = 0;
        }
        if (nl + na + nc != inflight) { cnt[CNT_ERR] = ERR_QUEUE_STATE; goto done; }
        if (inflight > cnt[CNT_MAX_INFLIGHT]) cnt[CNT_MAX_INFLIGHT] = inflight;
    }
done:
    free(q_look); free(q_adv); free(q_col);
}

/* Entry point used by oracle/driver.py for one worker's share of a batch. */
void oracle_run_batch(const int64_t *assigned, int64_t n_assigned, const OSlots *S, const OLib *L,
                      const OGeom *G, const OSrc *src, OLog *lg, OSites *sb, double *wbins, int32_t nbins,
                      int64_t *cnt, double *tm, const OParams *P) {
    if (P->history) run_history_batch(assigned, n_assigned, S, L, G, src, lg, sb, wbins, nbins, cnt, tm, P);
    else run_event_batch(assigned, n_assigned, S, L, G, src, lg, sb, wbins, nbins, cnt, tm, P);
}

/* K:1219-1223 */
void oracle_replay_into_bins(double *bins, const int32_t *binidx, const double *vals, int64_t n) {
    for (int64_t e = 0; e < n; ++e) bins[binidx[e]] += vals[e];
}
