// libemc.so: host side of the B200 transport engine and its C ABI (include/emc.h).
//
// One emc_ctx per GPU (one process per GPU under torch.distributed).  The
// context owns the device library (interleaved grid records + log-hash
// bracket table), the particle slots (SoA), the event queues, the fission
// bank and the contribution log, and drives the event loop of one batch:
//
//   source_init -> { [sort] -> lookup -> advance -> crossing | collision(+refill) }*
//   -> canonical bank sort -> (deterministic) log sort
//
// Reference: replication.py:114-142 (_run_worker_batch) and kernels.py:1092-1211.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/emc.h"
#include "emc_aux_kernels.cuh"
#include "emc_history.cuh"
#include "emc_kernels.cuh"
#include "emc_lookup_staged.cuh"

using namespace emc;

static thread_local std::string g_err;

#define EMC_TRY_CUDA(expr)                                                             \
    do {                                                                               \
        cudaError_t e_ = (expr);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            g_err = std::string(#expr) + ": " + cudaGetErrorString(e_);                \
            return EMC_E_CUDA;                                                         \
        }                                                                              \
    } while (0)

#define EMC_CHECK_LAUNCH(ctx)                                                          \
    do {                                                                               \
        (ctx)->launches++;                                                             \
        cudaError_t e_ = cudaGetLastError();                                           \
        if (e_ != cudaSuccess) {                                                       \
            g_err = std::string("kernel launch: ") + cudaGetErrorString(e_);           \
            return EMC_E_CUDA;                                                         \
        }                                                                              \
    } while (0)

static int fail_arg(const char* msg) { g_err = msg; return EMC_E_ARG; }

namespace {

// device buffer with typed pointer; realloc drops contents
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    int alloc(size_t count) {
        if (count <= n && p) return 0;
        if (p) cudaFree(p);
        p = nullptr; n = 0;
        if (count == 0) return 0;
        if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            g_err = "cudaMalloc failed (" + std::to_string(count * sizeof(T)) + " bytes)";
            return EMC_E_OOM;
        }
        n = count;
        return 0;
    }
    void release() { if (p) cudaFree(p); p = nullptr; n = 0; }
};

struct SiteBufs {
    DBuf<int64_t> parent; DBuf<int32_t> ord;
    DBuf<double> x, y, z, dx, dy, dz, E;
    int alloc(size_t cap) {
        int rc = 0;
        rc |= parent.alloc(cap); rc |= ord.alloc(cap);
        rc |= x.alloc(cap); rc |= y.alloc(cap); rc |= z.alloc(cap);
        rc |= dx.alloc(cap); rc |= dy.alloc(cap); rc |= dz.alloc(cap); rc |= E.alloc(cap);
        return rc ? EMC_E_OOM : 0;
    }
    DSites view() const {
        return DSites{parent.p, ord.p, x.p, y.p, z.p, dx.p, dy.p, dz.p, E.p, (int64_t)parent.n};
    }
    void release() {
        parent.release(); ord.release(); x.release(); y.release(); z.release();
        dx.release(); dy.release(); dz.release(); E.release();
    }
};

inline int grid_for(int64_t n, int block, int max_blocks)
{
    int64_t b = (n + block - 1) / block;
    if (b < 1) b = 1;
    return (int)std::min<int64_t>(b, max_blocks);
}

}  // namespace

struct emc_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;

    // library
    bool have_lib = false;
    DBuf<Rec> rec; DBuf<double> ch_s, nu; DBuf<int32_t> mat_off; DBuf<Comp> comp; DBuf<int32_t> hash;
    DBuf<int32_t> mat_group, grp_off; DBuf<NucRef> gnuc; DBuf<DD> ddT; DBuf<double> denS; DBuf<IvRec> iv; DBuf<int32_t> nsafe;
    int32_t n_groups = 0;
    DLib L{};
    // union-grid lookup backends (RunConfig.accel, emc_upload_union / emc_set_accel)
    DUnion U{};
    DBuf<double> u_grid, u_merged; DBuf<int32_t> u_hash, u_map;
    int32_t n_nuc = 0;
    int32_t n_materials = 0, max_comp = 0, n_entries = 0;
    double nu_max = 0.0;         // largest nu of the library (bounds the fission-site ordinal)
    int64_t lib_bytes = 0;

    // geometry
    bool have_geom = false;
    DBuf<double> zplanes; DBuf<int32_t> fuel_mats;
    DBuf<int32_t> pin_map; DBuf<double> pin_xy;
    DGeom G{};

    // extensions: fixed surface source, track-length mesh
    int32_t fixed_source = 0;
    double src_energy = 0.0;
    DBuf<double> mesh_acc;
    DMesh M{};

    // run configuration
    bool configured = false;
    emc_run_config cfg{};
    int64_t nslots = 0;
    int32_t nck = 0, n_bins = 0, kbin = 0, mat_bits = 1, grp_bits = 0, band_bits = 0, ebin_bits = 0;
    int32_t n_bands = 1, key_bits = 1, ebin_shift = 0;

    // particle slots
    // particle lines, double-buffered: after each lookup-queue sort the lines
    // are permuted into queue order (k_reorder), so every later sweep streams
    DBuf<PState> ps, ps2; DBuf<double> ckpt; DBuf<int32_t> iota;
    PState* ps_cur = nullptr;
    bool reorder = true;
    int lookup_block = 1024;
    bool staged = true;          // k_lookup_staged + energy-major sort (EMC_LOOKUP=plain: k_lookup)
    size_t lk_smem = 0;
    int lk_cfg = 2;              // chunk-synchronous staged lookup (tail queues) launch configuration (EMC_LK_CFG)
    bool lk_piped = true;        // chunk-pipelined staged lookup on sorted queues (EMC_LK_PIPED)
    int lk_pcfg = 1;             // its CTA configuration (EMC_LK_PCFG: 0 = 32 warps x 1, 1 = 16 warps x 2, 2 = 10 x 3)
    DSlots S{};
    bool ck_pmajor = false;      // sigma_t checkpoints particle-major (EMC_CK_PMAJOR)

    // queues + sort scratch
    DBuf<int32_t> qa, qb, qs, qc, qx;
    DBuf<uint32_t> keys_in, keys_out, keys_b;   // keys_in / keys_b: push-time keys paired with qa / qb
    DBuf<unsigned char> cub_tmp;

    // fission bank: raw appends + canonical (sorted) copy
    // two canonical-bank buffers: batch b reads bank[cur] (its source, when
    // local) and writes its own canonical bank into bank[1-cur]
    SiteBufs sites, banks[2];
    int cur_bank = 0;
    int64_t bank_n = 0;
    SiteBufs& bank() { return banks[cur_bank]; }
    DBuf<uint64_t> bkey_in, bkey_out; DBuf<int32_t> bidx_in, bidx_out;

    // contribution log
    DBuf<int64_t> lg_gid; DBuf<int32_t> lg_ord, lg_bin; DBuf<double> lg_val;
    int64_t log_n = 0;
    size_t log_want = 0;                  // capacity the next batch's log needs (presize_logs)
    DBuf<uint64_t> lkey_in, lkey_out; DBuf<double> lval_out;
    // the sorted log: CUB double-buffer mode ping-pongs (lkey_in, lkey_out) and
    // (lg_val, lval_out), so its scratch stays small at > 2^31 entries
    const uint64_t* lkey_sorted = nullptr; const double* lval_sorted = nullptr;
    int gid_bits = 1;

    // per batch
    DBuf<double> bins, bins_init, bins_out; DBuf<unsigned long long> cnt; DBuf<Ctl> ctl;
    Ctl* ctl_host = nullptr;
    DSrc src{};
    cudaEvent_t ev[16]{};
    // tail mode (EMC_TAIL_N, EMC_TAIL_K): queues below tail_n once the source is
    // exhausted run tail_k iterations per host round trip, unsorted
    int64_t tail_n = 262144;
    bool trace = getenv("EMC_TRACE") != nullptr;   // per-iteration queue length / lookup time on stderr
    int tail_k = 16;
    bool tail_plain = false;     // tail lookups with the one-particle-per-thread gather kernel (EMC_TAIL_LOOKUP=plain)
    int64_t tail_warp_n = 32768; // tail queues up to this length use the warp-per-particle lookup (EMC_TAIL_WARP_N)
    int64_t tail_sub_n = 131072; // ... up to this length 8 lanes per particle (EMC_TAIL_SUB_N)
    bool all_small = false;      // no composition group is staged (all < LK_MIN_NUC): the gather kernel serves
    // small-population finish (EMC_FINISH_N): a tail queue at most this long is
    // carried to death in one launch (k_finish: one thread per particle for
    // gather-lookup libraries; k_finish_warp: one warp per particle for staged
    // ones); -1 = by library (whole tail / 32768)
    int64_t finish_n = -1;
    bool finish_warp = false;    // EMC_FINISH_WARP=1: warp-per-particle finish for gather-lookup libraries too
    cudaEvent_t evt[4 * 32]{};
    bool ev_init = false;
};

// ------------------------------------------------------------------ misc ---

extern "C" const char* emc_last_error(void) { return g_err.c_str(); }
extern "C" int emc_abi_version(void) { return EMC_ABI_VERSION; }

extern "C" int emc_device_count(int* n)
{
    EMC_TRY_CUDA(cudaGetDeviceCount(n));
    return 0;
}

extern "C" int emc_create(int device, emc_ctx** out)
{
    if (!out) return fail_arg("emc_create: out is NULL");
    EMC_TRY_CUDA(cudaSetDevice(device));
    emc_ctx* c = new emc_ctx();
    c->device = device;
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    {
        uint64_t tab[2][64];
        lcg_gskip_table(tab);
        EMC_TRY_CUDA(cudaMemcpyToSymbol(c_gskip, tab, sizeof(tab)));
    }
    if (cudaMallocHost(&c->ctl_host, sizeof(Ctl)) != cudaSuccess) { delete c; g_err = "cudaMallocHost"; return EMC_E_CUDA; }
    if (c->ctl.alloc(1) || c->cnt.alloc(EMC_N_COUNTERS)) { delete c; return EMC_E_OOM; }
    for (auto& e : c->ev) cudaEventCreate(&e);
    for (auto& e : c->evt) cudaEventCreate(&e);
    if (const char* t = getenv("EMC_TAIL_N")) c->tail_n = std::max<int64_t>(0, atoll(t));
    if (const char* t = getenv("EMC_TAIL_K")) c->tail_k = std::max(1, std::min(32, atoi(t)));
    if (const char* t = getenv("EMC_TAIL_LOOKUP")) c->tail_plain = std::strcmp(t, "plain") == 0;
    if (const char* t = getenv("EMC_TAIL_WARP_N")) c->tail_warp_n = std::max<int64_t>(0, atoll(t));
    if (const char* t = getenv("EMC_TAIL_SUB_N")) c->tail_sub_n = std::max<int64_t>(0, atoll(t));
    if (const char* t = getenv("EMC_FINISH_N")) c->finish_n = std::max<int64_t>(0, atoll(t));
    if (const char* t = getenv("EMC_FINISH_WARP")) c->finish_warp = atoi(t) != 0;
    c->ev_init = true;
    *out = c;
    return 0;
}

extern "C" void emc_destroy(emc_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto* b : {&c->ckpt, &c->ch_s, &c->nu, &c->zplanes, &c->bins, &c->bins_init,
                    &c->bins_out, &c->lg_val, &c->lval_out})
        b->release();
    for (auto* b : {&c->mat_off, &c->hash, &c->fuel_mats, &c->qa, &c->qb, &c->qs, &c->qc, &c->qx,
                    &c->bidx_in, &c->bidx_out, &c->lg_ord, &c->lg_bin})
        b->release();
    c->ps.release(); c->ps2.release(); c->iota.release(); c->rec.release(); c->comp.release();
    c->mat_group.release(); c->grp_off.release(); c->gnuc.release(); c->ddT.release(); c->denS.release(); c->iv.release(); c->nsafe.release();
    c->keys_in.release(); c->keys_out.release(); c->keys_b.release(); c->cub_tmp.release();
    c->bkey_in.release(); c->bkey_out.release(); c->lkey_in.release(); c->lkey_out.release();
    c->lg_gid.release(); c->cnt.release(); c->ctl.release();
    c->sites.release(); c->banks[0].release(); c->banks[1].release();
    if (c->ctl_host) cudaFreeHost(c->ctl_host);
    if (c->ev_init) {
        for (auto& e : c->ev) cudaEventDestroy(e);
        for (auto& e : c->evt) cudaEventDestroy(e);
    }
    delete c;
}

extern "C" int emc_set_stream(emc_ctx* c, void* stream)
{
    if (!c) return fail_arg("null ctx");
    c->stream = (cudaStream_t)stream;
    return 0;
}

extern "C" int64_t emc_launch_count(emc_ctx* c) { return c ? c->launches : -1; }

// --------------------------------------------------------------- library ---

extern "C" int emc_upload_library(emc_ctx* c, const emc_library* lib)
{
    if (!c || !lib) return fail_arg("emc_upload_library: null argument");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    const int64_t nn = lib->n_nuclides, np = lib->n_points, nm = lib->n_materials, ne = lib->n_entries;
    if (nn < 1 || nm < 1 || np < 1) return fail_arg("empty library");
    if (np > INT32_MAX / 2 || ne > INT32_MAX / 2) { g_err = "library too large for 32-bit indices"; return EMC_E_RANGE; }
    for (int64_t i = 0; i < nn; ++i)
        if (lib->grid_off[i + 1] - lib->grid_off[i] < 1) return fail_arg("nuclide with an empty grid");

    // interleaved {E, t, c, f} records
    std::vector<Rec> hrec(np);
    for (int64_t i = 0; i < np; ++i) hrec[i] = Rec{lib->grids[i], lib->ch_t[i], lib->ch_c[i], lib->ch_f[i]};

    // composition entries, with den*nu formed exactly as the reference does
    std::vector<Comp> hcomp(std::max<int64_t>(ne, 1));
    std::vector<int32_t> hmo(nm + 1);
    int32_t maxc = 0;
    for (int64_t m = 0; m <= nm; ++m) hmo[m] = (int32_t)lib->mat_off[m];
    for (int64_t m = 0; m < nm; ++m) maxc = std::max<int32_t>(maxc, (int32_t)(lib->mat_off[m + 1] - lib->mat_off[m]));
    for (int64_t k = 0; k < ne; ++k) {
        int32_t nid = lib->mat_nuc[k];
        if (nid < 0 || nid >= nn) return fail_arg("composition references an unknown nuclide");
        volatile double dn = lib->mat_den[k] * lib->nu[nid];
        hcomp[k] = Comp{lib->mat_den[k], (double)dn, (int32_t)lib->grid_off[nid],
                        (int32_t)(lib->grid_off[nid + 1] - lib->grid_off[nid]), nid, 0};
    }

    // log-hash: bins are (bits(E) >> shift); 2^m bins per octave with 2^m >=
    // the densest grid's points per octave.
    double lo = lib->emin, hi = lib->emax;
    if (!(lo > 0.0) || !(hi >= lo)) return fail_arg("library energy bounds must be positive");
    int64_t gmax = 1;
    for (int64_t i = 0; i < nn; ++i) gmax = std::max<int64_t>(gmax, lib->grid_off[i + 1] - lib->grid_off[i]);
    double octaves = std::max(1.0, std::log2(hi / lo));
    int mbits = (int)std::ceil(std::log2(std::max(1.0, (double)gmax / octaves)));
    if (const char* hb = getenv("EMC_HASH_EXTRA_BITS")) mbits += atoi(hb);   // tuning knob
    mbits = std::min(std::max(mbits, 0), 16);
    int shift = 52 - mbits;
    uint64_t blo, bhi;
    std::memcpy(&blo, &lo, 8); std::memcpy(&bhi, &hi, 8);
    int64_t key_lo = (int64_t)(blo >> shift), key_hi = (int64_t)(bhi >> shift);
    int64_t nbins = key_hi - key_lo + 1;
    if (nbins * nn > (int64_t)1 << 31) { g_err = "hash table too large"; return EMC_E_RANGE; }
    std::vector<int32_t> hhash(nbins * nn);
    for (int64_t nid = 0; nid < nn; ++nid) {
        const double* gr = lib->grids + lib->grid_off[nid];
        int64_t G = lib->grid_off[nid + 1] - lib->grid_off[nid];
        int64_t j = 0;   // number of grid points <= current bin's lower edge
        for (int64_t b = 0; b < nbins; ++b) {
            uint64_t eb = (uint64_t)(key_lo + b) << shift;
            double edge;
            std::memcpy(&edge, &eb, 8);
            while (j < G && gr[j] <= edge) ++j;
            int64_t start = j - 1;                       // searchsorted(right) - 1
            if (start < 0) start = 0;
            if (b == 0) start = 0;
            if (G >= 2 && start > G - 2) start = G - 2;
            if (G < 2) start = 0;
            hhash[nid * nbins + b] = (int32_t)start;
        }
    }

    // composition groups: identical nuclide lists -> one group (see DLib)
    std::vector<int32_t> hgroup(nm), hgoff(1, 0);
    std::vector<NucRef> hgnuc;
    std::vector<std::vector<int32_t>> sigs;
    for (int64_t m = 0; m < nm; ++m) {
        std::vector<int32_t> sig(lib->mat_nuc + lib->mat_off[m], lib->mat_nuc + lib->mat_off[m + 1]);
        int32_t g = -1;
        for (size_t j = 0; j < sigs.size(); ++j) if (sigs[j] == sig) { g = (int32_t)j; break; }
        if (g < 0) {
            g = (int32_t)sigs.size();
            sigs.push_back(sig);
            for (int32_t nid : sig)
                hgnuc.push_back(NucRef{(int32_t)lib->grid_off[nid], (int32_t)(lib->grid_off[nid + 1] - lib->grid_off[nid]),
                                       (int32_t)(nid * nbins), nid});
            // staged groups are padded to whole pipeline stages with copies of
            // their first nuclide at zero density: den*t = +0 leaves every
            // running sum bit-identical, and the consumers need no bound checks
            if ((int32_t)sig.size() >= LK_MIN_NUC)
                while ((hgnuc.size() - hgoff.back()) % LK_G) hgnuc.push_back(hgnuc[hgoff.back()]);
            hgoff.push_back((int32_t)hgnuc.size());
        }
        hgroup[m] = g;
    }
    if (hgnuc.empty()) hgnuc.push_back(NucRef{0, 1, 0, 0});
    int32_t maxg = std::max(maxc, 1);          // longest (padded) group list
    for (size_t g = 0; g + 1 < hgoff.size(); ++g) maxg = std::max(maxg, hgoff[g + 1] - hgoff[g]);
    std::vector<DD> hdd((size_t)maxg * nm, DD{0.0, 0.0});
    for (int64_t m = 0; m < nm; ++m)
        for (int64_t k = lib->mat_off[m]; k < lib->mat_off[m + 1]; ++k)
            hdd[(size_t)(k - lib->mat_off[m]) * nm + m] = DD{hcomp[k].den, hcomp[k].dn};
    // staged lookup: densities as [stage][material][LK_G] blocks (one bulk copy per stage)
    const int64_t nstage = (maxg + LK_G - 1) / LK_G;
    std::vector<double> hden((size_t)nstage * nm * LK_DS, 0.0);
    for (int64_t m = 0; m < nm; ++m)
        for (int64_t k = lib->mat_off[m]; k < lib->mat_off[m + 1]; ++k) {
            const int64_t pos = k - lib->mat_off[m];
            double* e = &hden[((size_t)(pos / LK_G) * nm + m) * LK_DS + 2 * (pos % LK_G)];
            e[0] = hcomp[k].den;
            e[1] = hcomp[k].dn;      // den*nu exactly as the reference forms it (K:632)
        }
    const int32_t den_staged = (size_t)LK_D * lk_den_block((int)nm) <= (size_t)LK_DEN_BYTES_MAX;
    // nuclides whose grid lies where the staged lookup's guard-free division is exact
    std::vector<int32_t> hsafe(nn, 1);
    for (int64_t nid = 0; nid < nn; ++nid) {
        const double* gr = lib->grids + lib->grid_off[nid];
        const int64_t G = lib->grid_off[nid + 1] - lib->grid_off[nid];
        for (int64_t i = 0; i < G && hsafe[nid]; ++i) {
            if (!div_safe_range(gr[i])) hsafe[nid] = 0;
            if (i + 1 < G && !div_safe_range(gr[i + 1] - gr[i])) hsafe[nid] = 0;
        }
    }

    int rc = 0;
    rc |= c->mat_group.alloc(nm); rc |= c->grp_off.alloc(hgoff.size()); rc |= c->gnuc.alloc(hgnuc.size());
    rc |= c->ddT.alloc(hdd.size()); rc |= c->denS.alloc(hden.size()); rc |= c->iv.alloc(np); rc |= c->nsafe.alloc(nn);
    rc |= c->rec.alloc(np); rc |= c->ch_s.alloc(np); rc |= c->nu.alloc(nn); rc |= c->mat_off.alloc(nm + 1);
    rc |= c->comp.alloc(hcomp.size()); rc |= c->hash.alloc(hhash.size());
    if (rc) return EMC_E_OOM;
    EMC_TRY_CUDA(cudaMemcpy(c->rec.p, hrec.data(), np * sizeof(Rec), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->ch_s.p, lib->ch_s, np * sizeof(double), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->nu.p, lib->nu, nn * sizeof(double), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->mat_off.p, hmo.data(), (nm + 1) * sizeof(int32_t), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->comp.p, hcomp.data(), hcomp.size() * sizeof(Comp), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->hash.p, hhash.data(), hhash.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->mat_group.p, hgroup.data(), nm * sizeof(int32_t), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->grp_off.p, hgoff.data(), hgoff.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->gnuc.p, hgnuc.data(), hgnuc.size() * sizeof(NucRef), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->ddT.p, hdd.data(), hdd.size() * sizeof(DD), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->denS.p, hden.data(), hden.size() * sizeof(double), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->nsafe.p, hsafe.data(), nn * sizeof(int32_t), cudaMemcpyHostToDevice));
    {   // interval records (precomputed differences and reciprocals), built on the device
        DBuf<int64_t> goff;
        if (goff.alloc(nn + 1)) return EMC_E_OOM;
        EMC_TRY_CUDA(cudaMemcpy(goff.p, lib->grid_off, (nn + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
        dim3 grid((unsigned)std::min<int64_t>((gmax + 255) / 256, 64), (unsigned)nn);
        k_build_intervals<<<grid, 256>>>(c->rec.p, goff.p, (int32_t)nn, c->iv.p);
        EMC_TRY_CUDA(cudaGetLastError());
        EMC_TRY_CUDA(cudaDeviceSynchronize());
        goff.release();
    }
    c->n_groups = (int32_t)sigs.size();
    c->all_small = true;
    for (size_t g = 0; g < sigs.size(); ++g)
        if ((int32_t)sigs[g].size() >= LK_MIN_NUC) c->all_small = false;
    c->L = DLib{c->rec.p, c->ch_s.p, c->nu.p, c->mat_off.p, c->comp.p, c->hash.p, key_lo, (int32_t)nbins,
                shift, lo, hi, c->mat_group.p, c->grp_off.p, c->gnuc.p, c->ddT.p, (int32_t)nm, 0,
                c->iv.p, c->denS.p, den_staged, 0, c->nsafe.p};
    c->lk_smem = lk_pipe_offset((int)nm, den_staged) + sizeof(LkPipe);
    EMC_TRY_CUDA(lk_set_smem(c->lk_smem));
    if (const char* lc = getenv("EMC_LK_CFG")) c->lk_cfg = std::max(0, std::min(LK_NCFG - 1, atoi(lc)));
    c->n_materials = (int32_t)nm;
    c->n_entries = (int32_t)ne;
    c->max_comp = maxc;
    c->nu_max = 0.0;
    for (int64_t i = 0; i < nn; ++i) c->nu_max = std::max(c->nu_max, lib->nu[i]);
    c->lib_bytes = (int64_t)(np * (sizeof(Rec) + 8) + hcomp.size() * sizeof(Comp) + hhash.size() * 4);
    c->have_lib = true;
    c->n_nuc = (int32_t)nn;
    c->u_grid.release(); c->u_merged.release(); c->u_hash.release(); c->u_map.release();
    c->U = DUnion{};
    return 0;
}

extern "C" int emc_upload_geometry(emc_ctx* c, const emc_geometry* g)
{
    if (!c || !g) return fail_arg("emc_upload_geometry: null argument");
    if (g->n_axial < 1) return fail_arg("n_axial must be >= 1");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    if (c->zplanes.alloc(g->n_axial + 1) || c->fuel_mats.alloc(g->n_axial)) return EMC_E_OOM;
    EMC_TRY_CUDA(cudaMemcpy(c->zplanes.p, g->zplanes, (g->n_axial + 1) * 8, cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->fuel_mats.p, g->fuel_mats, g->n_axial * 4, cudaMemcpyHostToDevice));
    c->G = DGeom{g->radius, g->r2, g->half_pitch, g->height, (int32_t)g->n_axial, (int32_t)g->mod_mat,
                 c->zplanes.p, c->fuel_mats.p, 0, 0, 0, 0, 1, 0, 0.0, nullptr, nullptr};
    c->M.on = 0;
    c->n_bins = (int32_t)((g->n_axial + 1) * 5 + 1);
    c->kbin = c->n_bins - 1;
    c->have_geom = true;
    return 0;
}

extern "C" int emc_set_geometry_options(emc_ctx* c, int32_t slab, int32_t vacuum)
{
    if (!c || !c->have_geom) return fail_arg("emc_set_geometry_options: upload the geometry first");
    c->G.slab = slab ? 1 : 0;
    c->G.vacuum = vacuum ? 1 : 0;
    return 0;
}

extern "C" int emc_set_lattice(emc_ctx* c, int32_t n, double pitch, const int32_t* pin_map)
{
    if (!c || !c->have_geom) return fail_arg("emc_set_lattice: upload the geometry first");
    if (n <= 1) { c->G.lat_n = 1; c->G.n_pins = 0; return 0; }
    if (!pin_map || !(pitch > 0.0)) return fail_arg("emc_set_lattice: bad arguments");
    if (!(2.0 * c->G.radius < pitch)) return fail_arg("emc_set_lattice: pins must fit their cells");
    if (std::fabs(n * pitch - 2.0 * c->G.hp) > 1e-12 * n * pitch)
        return fail_arg("emc_set_lattice: the box half-width must be n*pitch/2");
    std::vector<double> xy;
    for (int32_t j = 0; j < n; ++j)
        for (int32_t i = 0; i < n; ++i)
            if (pin_map[j * n + i]) {     // centres exactly as lattice_cell() forms them
                xy.push_back(-c->G.hp + ((double)i + 0.5) * pitch);
                xy.push_back(-c->G.hp + ((double)j + 0.5) * pitch);
            }
    if (xy.empty()) return fail_arg("emc_set_lattice: no fuel pins");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    // device copy: one bit per cell (the 323 x 323 HM core lattice is 13 KB,
    // L1-resident, instead of 417 KB of int32)
    const int64_t nw = ((int64_t)n * n + 31) / 32;
    if (c->pin_map.alloc(nw) || c->pin_xy.alloc(xy.size())) return EMC_E_OOM;
    std::vector<int32_t> pm((size_t)nw, 0);
    for (int64_t k = 0; k < (int64_t)n * n; ++k)
        if (pin_map[k]) pm[(size_t)(k >> 5)] |= (int32_t)(1u << (k & 31));
    EMC_TRY_CUDA(cudaMemcpy(c->pin_map.p, pm.data(), pm.size() * 4, cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->pin_xy.p, xy.data(), xy.size() * 8, cudaMemcpyHostToDevice));
    c->G.lat_n = n; c->G.n_pins = (int32_t)(xy.size() / 2); c->G.pitch = pitch;
    c->G.pin_map = c->pin_map.p; c->G.pin_xy = c->pin_xy.p;
    return 0;
}

extern "C" int emc_set_fixed_source(emc_ctx* c, int32_t enabled, double energy)
{
    if (!c) return fail_arg("null ctx");
    if (enabled && !(energy >= 0.0)) return fail_arg("fixed source energy must be >= 0 (0: fission spectrum)");
    c->fixed_source = enabled ? 1 : 0;
    c->src_energy = energy;
    return 0;
}

extern "C" int emc_set_mesh(emc_ctx* c, int32_t nx, int32_t ny, int32_t nz)
{
    if (!c || !c->have_geom) return fail_arg("emc_set_mesh: upload the geometry first");
    if (nx <= 0 || ny <= 0 || nz <= 0) { c->M.on = 0; return 0; }
    const int64_t cells = (int64_t)nx * ny * nz;
    if (cells > (int64_t)1 << 28) return fail_arg("mesh too large");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    if (c->mesh_acc.alloc(2 * cells)) return EMC_E_OOM;
    EMC_TRY_CUDA(cudaMemset(c->mesh_acc.p, 0, 2 * cells * sizeof(double)));
    const double hp = c->G.hp, h = c->G.height;
    c->M = DMesh{c->mesh_acc.p, nx, ny, nz, 1, -hp, -hp, 0.0, (2.0 * hp) / nx, (2.0 * hp) / ny, h / nz};
    return 0;
}

extern "C" int emc_mesh_device(emc_ctx* c, double** ptr, int64_t* n)
{
    if (!c || !ptr || !n) return fail_arg("emc_mesh_device: null argument");
    *ptr = c->M.on ? c->M.acc : nullptr;
    *n = c->M.on ? 2 * (int64_t)c->M.nx * c->M.ny * c->M.nz : 0;
    return 0;
}

// -------------------------------------------------------------- configure ---

static int alloc_sites(emc_ctx* c, size_t cap)
{
    // never touches banks[cur_bank]: it may be this batch's source
    if (c->sites.alloc(cap) || c->banks[1 - c->cur_bank].alloc(cap)) return EMC_E_OOM;
    if (c->bkey_in.alloc(cap) || c->bkey_out.alloc(cap) || c->bidx_in.alloc(cap) || c->bidx_out.alloc(cap))
        return EMC_E_OOM;
    return 0;
}

static int alloc_logs(emc_ctx* c, size_t cap)
{
    if (c->lg_gid.alloc(cap) || c->lg_ord.alloc(cap) || c->lg_bin.alloc(cap) || c->lg_val.alloc(cap)) return EMC_E_OOM;
    if (c->lkey_in.alloc(cap) || c->lkey_out.alloc(cap) || c->lval_out.alloc(cap)) return EMC_E_OOM;
    return 0;
}

extern "C" int emc_configure(emc_ctx* c, const emc_run_config* cfg)
{
    if (!c || !cfg) return fail_arg("emc_configure: null argument");
    if (!c->have_lib || !c->have_geom) return fail_arg("upload library and geometry before emc_configure");
    if (cfg->n_assigned < 1 || cfg->max_in_flight < 1 || cfg->sort_every < 1) return fail_arg("bad run config");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    c->cfg = *cfg;
    int64_t nslots = std::max<int64_t>(1, std::min<int64_t>(cfg->max_in_flight, cfg->n_assigned));
    if (nslots > INT32_MAX / 2) { g_err = "max_in_flight too large"; return EMC_E_RANGE; }
    c->nslots = nslots;
    c->nck = cfg->fused ? std::max(0, (c->max_comp - 1) / kCkptStride) : 0;
    int rc = 0;
    rc |= c->ps.alloc(nslots);
    if (const char* lb = getenv("EMC_LOOKUP_BLOCK")) c->lookup_block = atoi(lb);
    c->staged = c->U.accel == 0;      // the union backends use the one-thread-per-particle gather
    if (const char* lk = getenv("EMC_LOOKUP")) c->staged = c->staged && std::strcmp(lk, "plain") != 0;
    c->lk_piped = true;
    if (const char* lp = getenv("EMC_LK_PIPED")) c->lk_piped = atoi(lp) != 0;
    c->lk_pcfg = 1;
    if (const char* lp = getenv("EMC_LK_PCFG")) c->lk_pcfg = std::max(0, std::min(LK_NPCFG - 1, atoi(lp)));
    const char* ro = getenv("EMC_REORDER");
    c->reorder = !(ro && ro[0] == '0');
    if (c->reorder) rc |= c->ps2.alloc(nslots);
    rc |= c->iota.alloc(nslots);
    // sigma_t checkpoint layout (DSlots): row-major [nck][nslots] or, with
    // EMC_CK_PMAJOR=1, particle-major [nslots][nck rounded up to 4] (32-byte rows)
    const char* pm = getenv("EMC_CK_PMAJOR");
    c->ck_pmajor = pm && pm[0] == '1';
    const int64_t nck_pad = c->ck_pmajor ? ((int64_t)c->nck + 3) / 4 * 4 : c->nck;
    rc |= c->ckpt.alloc(std::max<int64_t>(1, nck_pad * nslots));
    for (auto* b : {&c->qa, &c->qb, &c->qs, &c->qc, &c->qx})
        rc |= b->alloc(nslots);
    rc |= c->keys_in.alloc(nslots); rc |= c->keys_out.alloc(nslots); rc |= c->keys_b.alloc(nslots);
    rc |= c->bins.alloc(c->n_bins); rc |= c->bins_init.alloc(c->n_bins); rc |= c->bins_out.alloc(c->n_bins);
    if (rc) return EMC_E_OOM;
    if (rc) return EMC_E_OOM;
    {
        std::vector<int32_t> h(nslots);
        for (int64_t i = 0; i < nslots; ++i) h[i] = (int32_t)i;
        EMC_TRY_CUDA(cudaMemcpy(c->iota.p, h.data(), nslots * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    c->ps_cur = c->ps.p;
    c->S = DSlots{c->ps_cur, c->ckpt.p, nslots, c->nck, c->ck_pmajor ? (int32_t)nck_pad : 1,
                  c->ck_pmajor ? (int64_t)1 : nslots};
    // fission bank: reference starts at n_assigned*6+1024 (R:92); ~1 site per
    // source particle is typical, so start at 2x and grow on overflow.
    if ((rc = alloc_sites(c, (size_t)(cfg->n_assigned * 2 + 4096)))) return rc;
    // both canonical banks up front (a run starts without a live source bank)
    if (c->banks[c->cur_bank].alloc(c->sites.parent.n)) return EMC_E_OOM;
    c->log_want = 0;
    if (cfg->use_logs) {
        // an unscored batch logs ~1 k-bin entry per collision (~4 per history at
        // C4); later batches are presized from the previous one (log_want), so
        // the log never holds the 64 entries per particle a scored batch may
        // need before one has run (48 B per entry: ~120 GB at 40M particles)
        if ((rc = alloc_logs(c, (size_t)(cfg->n_assigned * 8 + 4096)))) return rc;
    }
    // lookup sort key (32 bits): group | energy band | material | energy bin
    // (see k_sort_keys).  EMC_SORT_BANDS overrides the band count (1 = pure
    // material-major order).
    {
        auto bits = [](int64_t v) { int b = 0; while (((int64_t)1 << b) < v) ++b; return b; };
        int nb = 64;
        if (const char* e = getenv("EMC_SORT_BANDS")) nb = std::max(1, atoi(e));
        if (c->staged) nb = 1;
        c->n_bands = nb;
        c->grp_bits = bits(c->n_groups);
        c->band_bits = bits(nb);
        if (c->staged) {     // energy-major key: band field = fine energy bits (EMC_SORT_FINE)
            c->band_bits = 5;
            if (const char* e = getenv("EMC_SORT_FINE")) c->band_bits = std::max(0, std::min(12, atoi(e)));
        }
        c->mat_bits = bits(c->n_materials);
        if (c->staged) if (const char* e = getenv("EMC_SORT_MAT")) if (atoi(e) == 0) c->mat_bits = 0;
        c->ebin_bits = bits(c->L.nbins);
        int total = c->grp_bits + c->band_bits + c->mat_bits + c->ebin_bits;
        if (total > 32) {            // drop fine-energy bits first (order stays valid)
            c->ebin_bits = std::max(0, c->ebin_bits - (total - 32));
            total = c->grp_bits + c->band_bits + c->mat_bits + c->ebin_bits;
        }
        if (total > 32) { g_err = "too many materials/groups for the 32-bit sort key"; return EMC_E_RANGE; }
        c->key_bits = total;
        c->ebin_shift = bits(c->L.nbins) - c->ebin_bits;
    }
    int gidb = 1;
    while (((int64_t)1 << gidb) < cfg->n_assigned) ++gidb;
    c->gid_bits = gidb;
    int bb = 1;
    while ((1 << bb) < c->n_bins) ++bb;
    if (bb + gidb + 17 > 64) { g_err = "deterministic log key exceeds 64 bits"; return EMC_E_RANGE; }
    // CUB scratch, sized up front for the largest sorts we run (queue keys over
    // the slots; 32- and 64-bit bank keys over the site capacity), so no batch
    // pays a mid-run reallocation
    size_t t1 = 0, t2 = 0, t3 = 0;
    const int64_t scap = (int64_t)c->sites.parent.n;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)std::max<int64_t>(nslots, scap), 0, 32);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint64_t*)nullptr, (uint64_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)scap, 0, 64);
    if (cfg->use_logs) {
        cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
        cub::DoubleBuffer<double> dv(nullptr, nullptr);
        cub::DeviceRadixSort::SortPairs(nullptr, t3, dk, dv, (int64_t)c->lg_gid.n, 0, 64);
    }
    if (c->cub_tmp.alloc(std::max<size_t>(std::max(t1, std::max(t2, t3)), 1))) return EMC_E_OOM;
    c->bank_n = 0;
    c->src = DSrc{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0.0, 0};
    c->configured = true;
    return 0;
}

extern "C" int emc_set_source_local(emc_ctx* c, double u)
{
    if (!c || !c->configured) return fail_arg("not configured");
    if (c->bank_n < 1) return fail_arg("no local bank to resample");
    SiteBufs& b = c->bank();
    c->src = DSrc{b.x.p, b.y.p, b.z.p, b.dx.p, b.dy.p, b.dz.p, b.E.p, c->bank_n, u, 0};
    return 0;
}

extern "C" int emc_set_source_device(emc_ctx* c, const void* const ptrs[7], int64_t n, double u)
{
    if (!c || !c->configured || !ptrs) return fail_arg("emc_set_source_device: bad arguments");
    if (n < 1) return fail_arg("empty source bank");
    c->src = DSrc{(const double*)ptrs[0], (const double*)ptrs[1], (const double*)ptrs[2], (const double*)ptrs[3],
                  (const double*)ptrs[4], (const double*)ptrs[5], (const double*)ptrs[6], n, u, 0};
    return 0;
}

extern "C" int emc_set_source_window(emc_ctx* c, const void* const ptrs[7], int64_t n, double u, int64_t lo)
{
    int rc = emc_set_source_device(c, ptrs, n, u);
    if (rc) return rc;
    if (lo < 0 || lo >= n) return fail_arg("emc_set_source_window: lo outside the bank");
    c->src.lo = lo;
    return 0;
}

// ----------------------------------------------------------------- batch ---

static int sort_cub(emc_ctx* c, const uint32_t* kin, uint32_t* kout, const int32_t* vin, int32_t* vout, int n,
                    int end_bit)
{
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, kin, kout, vin, vout, n, 0, end_bit, c->stream);
    if (need > c->cub_tmp.n && c->cub_tmp.alloc(need)) return EMC_E_OOM;
    EMC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, need, kin, kout, vin, vout, n, 0, end_bit, c->stream));
    c->launches += 4;
    return 0;
}

template <class K, class V>
static int sort_cub64(emc_ctx* c, const K* kin, K* kout, const V* vin, V* vout, int64_t n, int end_bit)
{
    size_t need = 0;
    // 64-bit item count: a deterministic-mode contribution log passes 2^31
    // entries at ~40M histories per rank (CUB's NumItemsT is templated)
    cub::DeviceRadixSort::SortPairs(nullptr, need, kin, kout, vin, vout, n, 0, end_bit, c->stream);
    if (need > c->cub_tmp.n && c->cub_tmp.alloc(need)) return EMC_E_OOM;
    EMC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, need, kin, kout, vin, vout, n, 0, end_bit,
                                                 c->stream));
    c->launches += (end_bit + 7) / 8;
    return 0;
}

// layout of the staged path's sort key (lookup_key): group | ebin | material | fine energy bits
static LkKeys lk_keys(const emc_ctx* c, const uint32_t* keys)
{
    LkKeys K;
    K.keys = keys;
    K.eb_shift = c->mat_bits + c->band_bits;
    K.grp_shift = c->ebin_bits + K.eb_shift;
    K.eb_mask = c->ebin_bits ? (uint32_t)((1ull << c->ebin_bits) - 1) : 0u;
    K.ebin_shift = c->ebin_shift;
    return K;
}

// grow the contribution log (and the CUB scratch of its sort) to c->log_want
static int presize_logs(emc_ctx* c)
{
    const size_t want = c->log_want;
    if (!c->cfg.use_logs || want <= c->lg_gid.n) return 0;
    // only when the larger log fits next to everything else (48 B per entry);
    // otherwise keep the current one: the next batch grows-and-reruns if needed
    size_t free_b = 0, total_b = 0;
    EMC_TRY_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if ((want - c->lg_gid.n) * 48 + ((size_t)1 << 30) > free_b) return 0;
    c->lg_gid.release(); c->lg_ord.release(); c->lg_bin.release(); c->lg_val.release();
    c->lkey_in.release(); c->lkey_out.release(); c->lval_out.release();
    if (int rc = alloc_logs(c, want)) return rc;
    size_t need = 0;
    cub::DoubleBuffer<uint64_t> dk(c->lkey_in.p, c->lkey_out.p);
    cub::DoubleBuffer<double> dv(c->lg_val.p, c->lval_out.p);
    cub::DeviceRadixSort::SortPairs(nullptr, need, dk, dv, (int64_t)want, 0, 64, c->stream);
    if (need > c->cub_tmp.n && c->cub_tmp.alloc(need)) return EMC_E_OOM;
    return 0;
}

static int bits_for(int64_t v)
{
    int b = 1;
    while (b < 63 && ((int64_t)1 << b) <= v) ++b;
    return b;
}

// one attempt at a batch; returns 0 and fills res (res->error may be set)
static int run_batch_once(emc_ctx* c, const emc_batch_args* a, emc_batch_result* res)
{
    const emc_run_config& cf = c->cfg;
    cudaStream_t st = c->stream;
    BatchP bp{};
    bp.seed = cf.seed & kLcgMask;
    bp.batch = a->batch; bp.pmax = cf.particles_per_batch; bp.g_lo = cf.gid_lo; bp.n_assigned = cf.n_assigned;
    bp.perturb_gid = cf.perturb_gid; bp.alpha = cf.alpha; bp.fission_t = cf.fission_t; bp.k_run = a->k_run;
    bp.fused = cf.fused; bp.score = a->score; bp.use_logs = cf.use_logs; bp.batch0 = a->batch0;
    bp.kbin = c->kbin; bp.history = cf.history;
    bp.fixed_source = c->fixed_source; bp.src_energy = c->src_energy;
    bp.seed_b = lcg_skip(bp.seed, (uint64_t)bp.batch * (uint64_t)bp.pmax * (uint64_t)kStride);
    if (!a->batch0 && !c->fixed_source && (c->src.n < 1 || !c->src.x))
        return fail_arg("batch > 0 needs a source bank (emc_set_source_*)");

    DSites sv = c->sites.view();
    DLog lg{c->lg_gid.p, c->lg_ord.p, c->lg_bin.p, c->lg_val.p, (int64_t)c->lg_gid.n};

    EMC_TRY_CUDA(cudaMemsetAsync(c->cnt.p, 0, EMC_N_COUNTERS * sizeof(unsigned long long), st));
    EMC_TRY_CUDA(cudaMemsetAsync(c->bins.p, 0, c->n_bins * sizeof(double), st));
    if (c->M.on)
        EMC_TRY_CUDA(cudaMemsetAsync(c->M.acc, 0, 2 * (size_t)c->M.nx * c->M.ny * c->M.nz * sizeof(double), st));
    Ctl z{};
    const int64_t n0 = std::min<int64_t>(c->nslots, cf.n_assigned);
    z.cursor = (unsigned long long)n0;
    EMC_TRY_CUDA(cudaMemcpyAsync(c->ctl.p, &z, sizeof(Ctl), cudaMemcpyHostToDevice, st));

    int64_t host_cnt[EMC_N_COUNTERS] = {0};
    double tm[4] = {0, 0, 0, 0};
    int64_t iterations = 0;
    const int BLK = 256;
    const int maxb = c->sm_count * 16;

    if (cf.history) {
        // history executor: one thread per in-flight history (K:1043-1089)
        z.cursor = 0;
        EMC_TRY_CUDA(cudaMemcpyAsync(c->ctl.p, &z, sizeof(Ctl), cudaMemcpyHostToDevice, st));
        EMC_TRY_CUDA(cudaEventRecord(c->ev[0], st));
        int64_t nthr = n0;
        k_history<<<(unsigned)((nthr + 127) / 128), 128, 0, st>>>(bp, c->L, c->G, c->src, c->S, lg, sv, c->bins.p,
                                                                   c->ctl.p, c->cnt.p, nthr, c->M);
        EMC_CHECK_LAUNCH(c);
        EMC_TRY_CUDA(cudaEventRecord(c->ev[1], st));
        EMC_TRY_CUDA(cudaMemcpyAsync(c->ctl_host, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        EMC_TRY_CUDA(cudaStreamSynchronize(st));
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
        tm[0] = ms * 1e-3;
        host_cnt[CNT_MAX_INFLIGHT] = nthr;
        iterations = 1;
    } else {
        int32_t* cur = c->qa.p;
        int32_t* nxt = c->qb.p;
        // push-time sort keys (staged lookup's energy-major key), paired with the queues
        uint32_t* kcur = c->keys_in.p;
        uint32_t* knxt = c->keys_b.p;
        auto qk = [&](uint32_t* k) {
            return QKeys{c->staged ? k : nullptr, c->ebin_bits, c->ebin_shift, c->mat_bits, c->band_bits};
        };
        EMC_TRY_CUDA(cudaEventRecord(c->ev[5], st));
        k_source_init<<<grid_for(n0, BLK, maxb), BLK, 0, st>>>(bp, c->L, c->G, c->src, c->S, (int32_t)n0, cur,
                                                               c->ctl.p, c->cnt.p, qk(kcur));
        EMC_CHECK_LAUNCH(c);
        EMC_TRY_CUDA(cudaEventRecord(c->ev[6], st));
        EMC_TRY_CUDA(cudaMemcpyAsync(c->ctl_host, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        EMC_TRY_CUDA(cudaStreamSynchronize(st));
        if (c->trace) {
            float sm = 0;
            cudaEventElapsedTime(&sm, c->ev[5], c->ev[6]);
            std::fprintf(stderr, "emc-trace source_init_ms %.4f n0 %lld\n", sm, (long long)n0);
        }
        int64_t nL = c->ctl_host->nL2;
        int64_t look_inv = 0, tail_blocks = 0;
        float ms;
        while (nL > 0 && c->ctl_host->err == 0) {
            const int64_t fin_n = c->finish_n >= 0 ? c->finish_n : (c->all_small ? c->tail_n : 32768);
            if (nL <= fin_n && c->ctl_host->cursor >= (unsigned long long)cf.n_assigned) {
                // small population: finish every remaining history in one launch
                EMC_TRY_CUDA(cudaEventRecord(c->ev[0], st));
                if (c->all_small && !c->finish_warp) {   // gather-lookup library: one thread per particle
                    const int fb = nL <= 64LL * c->sm_count ? 32 : nL <= 128LL * c->sm_count ? 64 : 128;
                    k_finish<<<(unsigned)((nL + fb - 1) / fb), fb, 0, st>>>(cur, nL, bp, c->L, c->G, c->S, lg, sv,
                                                                            c->bins.p, c->ctl.p, c->cnt.p, c->M);
                }
                else                  // staged library: one warp per particle (warp-cooperative lookups)
                    k_finish_warp<<<(unsigned)std::min<int64_t>((nL + 3) / 4, (int64_t)c->sm_count * 16), 128, 0,
                                    st>>>(cur, nL, bp, c->L, c->G, c->S, lg, sv, c->bins.p, c->ctl.p, c->cnt.p, c->M);
                EMC_CHECK_LAUNCH(c);
                EMC_TRY_CUDA(cudaEventRecord(c->ev[1], st));
                EMC_TRY_CUDA(cudaMemsetAsync(&c->ctl.p->nL2, 0, sizeof(unsigned), st));
                EMC_TRY_CUDA(cudaMemcpyAsync(c->ctl_host, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
                EMC_TRY_CUDA(cudaStreamSynchronize(st));
                cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
                tm[0] += ms * 1e-3;
                host_cnt[CNT_INV_LOOKUP] += 1; host_cnt[CNT_INV_ADVANCE] += 1; host_cnt[CNT_INV_COLLISION] += 1;
                iterations += 1;
                nL = 0;
                break;
            }
            if (nL <= c->tail_n && c->ctl_host->cursor >= (unsigned long long)cf.n_assigned) {
                // tail mode: tail_k iterations back to back, queue lengths on the device
                const int K = c->tail_k;
                const unsigned gl = grid_for(nL, BLK, maxb);
                for (int k = 0; k < K; ++k) {
                    k_tail_begin<<<1, 1, 0, st>>>(c->ctl.p, c->cnt.p);
                    EMC_CHECK_LAUNCH(c);
                    EMC_TRY_CUDA(cudaEventRecord(c->evt[4 * k], st));
                    if (c->U.accel) {
                        if (c->U.accel == 2)
                            k_lookup_union<true><<<gl, 256, 0, st>>>(cur, (int32_t)nL, c->L, c->U, c->S, cf.fused,
                                                                     c->cnt.p, &c->ctl.p->nLcur);
                        else
                            k_lookup_union<false><<<gl, 256, 0, st>>>(cur, (int32_t)nL, c->L, c->U, c->S, cf.fused,
                                                                      c->cnt.p, &c->ctl.p->nLcur);
                        EMC_TRY_CUDA(cudaGetLastError());
                    } else if (nL <= c->tail_warp_n) {
                        // sparse tail: one warp per particle (latency of one fold, not of 272 gathers)
                        k_lookup_warp<32><<<grid_for(nL * 32, 256, 8 * c->sm_count), 256, 0, st>>>(
                            cur, (int32_t)nL, c->L, c->S, cf.fused, c->cnt.p, &c->ctl.p->nLcur);
                        EMC_TRY_CUDA(cudaGetLastError());
                    } else if (nL <= c->tail_sub_n) {
                        // mid-size tail: 8 lanes per particle
                        k_lookup_warp<8><<<grid_for(nL * 8, 256, 8 * c->sm_count), 256, 0, st>>>(
                            cur, (int32_t)nL, c->L, c->S, cf.fused, c->cnt.p, &c->ctl.p->nLcur);
                        EMC_TRY_CUDA(cudaGetLastError());
                    } else if (c->tail_plain || c->all_small) {
                        k_lookup<256><<<gl, 256, 0, st>>>(cur, (int32_t)nL, c->L, c->S, cf.fused, c->cnt.p,
                                                          &c->ctl.p->nLcur);
                        EMC_TRY_CUDA(cudaGetLastError());
                    } else {
                        EMC_TRY_CUDA(lk_launch<0>(c->lk_cfg, c->L, cur, nL, c->S, cf.fused, c->cnt.p, nullptr,
                                                  nullptr, nullptr, c->sm_count, c->lk_smem, st, &c->ctl.p->nLcur));
                    }
                    c->launches += 1;
                    EMC_TRY_CUDA(cudaEventRecord(c->evt[4 * k + 1], st));
                    k_advance<<<gl, BLK, 0, st>>>(cur, (int32_t)nL, bp, c->L, c->G, c->S, lg, c->bins.p, c->qc.p,
                                                  c->qx.p, c->ctl.p, c->cnt.p, c->M, &c->ctl.p->nLcur, nxt, qk(knxt));
                    EMC_CHECK_LAUNCH(c);
                    if (c->G.vacuum) {
                        k_crossing<<<gl, BLK, 0, st>>>(c->qx.p, &c->ctl.p->nX, bp, c->L, c->G, c->src, c->S, nxt,
                                                       c->ctl.p, c->cnt.p, qk(knxt));
                        EMC_CHECK_LAUNCH(c);
                    }
                    EMC_TRY_CUDA(cudaEventRecord(c->evt[4 * k + 2], st));
                    k_collision<<<gl, BLK, 0, st>>>(c->qc.p, &c->ctl.p->nC, bp, c->L, c->G, c->src, c->S, lg, sv,
                                                    c->bins.p, nxt, c->ctl.p, c->cnt.p, qk(knxt));
                    EMC_CHECK_LAUNCH(c);
                    k_tail_end<<<1, 1, 0, st>>>(c->ctl.p, c->cnt.p);
                    EMC_CHECK_LAUNCH(c);
                    EMC_TRY_CUDA(cudaEventRecord(c->evt[4 * k + 3], st));
                    std::swap(cur, nxt);
                    std::swap(kcur, knxt);
                }
                EMC_TRY_CUDA(cudaMemcpyAsync(c->ctl_host, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
                EMC_TRY_CUDA(cudaStreamSynchronize(st));
                for (int k = 0; k < K; ++k) {
                    cudaEventElapsedTime(&ms, c->evt[4 * k], c->evt[4 * k + 1]); tm[0] += ms * 1e-3;
                    cudaEventElapsedTime(&ms, c->evt[4 * k + 1], c->evt[4 * k + 2]); tm[1] += ms * 1e-3;
                    cudaEventElapsedTime(&ms, c->evt[4 * k + 2], c->evt[4 * k + 3]); tm[2] += ms * 1e-3;
                }
                iterations += K;
                tail_blocks++;
                nL = c->ctl_host->nL2;
                continue;
            }
            const int32_t* q = cur;
            EMC_TRY_CUDA(cudaMemsetAsync(&c->ctl.p->nL2, 0, (char*)(&c->ctl.p->nX + 1) - (char*)&c->ctl.p->nL2, st));
            bool do_sort = cf.sort_enabled && nL > 1 && (look_inv % cf.sort_every) == 0;
            EMC_TRY_CUDA(cudaEventRecord(c->ev[0], st));
            if (do_sort) {
                if (!c->staged) {     // the staged path's keys were written when the queue was pushed
                    k_sort_keys<false><<<grid_for(nL, BLK, 1 << 30), BLK, 0, st>>>(
                        cur, (int32_t)nL, c->ps_cur, c->L, kcur, c->ebin_bits, c->ebin_shift, c->mat_bits,
                        c->band_bits, c->n_bands);
                    EMC_CHECK_LAUNCH(c);
                }
                int rc = sort_cub(c, kcur, c->keys_out.p, cur, c->qs.p, (int)nL, c->key_bits);
                if (rc) return rc;
                q = c->qs.p;
                host_cnt[CNT_SORTS] += 1;
                if (c->reorder && (!c->staged || c->all_small)) {
                    PState* dst = c->ps_cur == c->ps.p ? c->ps2.p : c->ps.p;
                    k_reorder<<<grid_for(nL, BLK, 1 << 30), BLK, 0, st>>>(c->qs.p, (int32_t)nL, c->ps_cur, dst);
                    EMC_CHECK_LAUNCH(c);
                    c->ps_cur = dst;
                    c->S.ps = dst;
                    q = c->iota.p;
                }
            }
            look_inv++;
            EMC_TRY_CUDA(cudaEventRecord(c->ev[1], st));
            if (c->staged && !c->all_small) {
                // the staged lookup moves the lines into sorted order itself (fused reorder)
                PState* rdst = nullptr;
                if (do_sort && c->reorder) rdst = c->ps_cur == c->ps.p ? c->ps2.p : c->ps.p;
                if (do_sort && c->lk_piped)
                    EMC_TRY_CUDA(lk_launch_piped<0>(c->L, q, nL, c->S, cf.fused, c->cnt.p, nullptr, nullptr, nullptr,
                                                    c->sm_count, c->lk_smem, st, rdst, lk_keys(c, c->keys_out.p),
                                                    c->lk_pcfg));
                else
                    EMC_TRY_CUDA(lk_launch<0>(c->lk_cfg, c->L, q, nL, c->S, cf.fused, c->cnt.p, nullptr, nullptr,
                                              nullptr, c->sm_count, c->lk_smem, st, nullptr, rdst));
                if (rdst) {
                    c->ps_cur = rdst;
                    c->S.ps = rdst;
                    q = c->iota.p;
                }
            } else if (c->U.accel == 2) {
                k_lookup_union<true><<<grid_for(nL, 256, maxb), 256, 0, st>>>(q, (int32_t)nL, c->L, c->U, c->S,
                                                                             cf.fused, c->cnt.p, nullptr);
            } else if (c->U.accel == 1) {
                k_lookup_union<false><<<grid_for(nL, 256, maxb), 256, 0, st>>>(q, (int32_t)nL, c->L, c->U, c->S,
                                                                              cf.fused, c->cnt.p, nullptr);
            } else switch (c->lookup_block) {
            case 1024:
                k_lookup<1024><<<grid_for(nL, 1024, c->sm_count), 1024, 0, st>>>(q, (int32_t)nL, c->L, c->S,
                                                                                 cf.fused, c->cnt.p);
                break;
            case 512:
                k_lookup<512><<<grid_for(nL, 512, 2 * c->sm_count), 512, 0, st>>>(q, (int32_t)nL, c->L, c->S,
                                                                                  cf.fused, c->cnt.p);
                break;
            default:
                k_lookup<256><<<grid_for(nL, 256, maxb), 256, 0, st>>>(q, (int32_t)nL, c->L, c->S, cf.fused,
                                                                       c->cnt.p);
            }
            EMC_CHECK_LAUNCH(c);
            EMC_TRY_CUDA(cudaEventRecord(c->ev[2], st));
            k_advance<<<grid_for(nL, BLK, maxb), BLK, 0, st>>>(q, (int32_t)nL, bp, c->L, c->G, c->S, lg, c->bins.p,
                                                              c->qc.p, c->qx.p, c->ctl.p, c->cnt.p, c->M, nullptr, nxt,
                                                              qk(knxt));
            EMC_CHECK_LAUNCH(c);
            if (c->G.vacuum) {       // leakage: end and refill (reflective problems cross inside k_advance)
                k_crossing<<<grid_for(nL, BLK, maxb), BLK, 0, st>>>(c->qx.p, &c->ctl.p->nX, bp, c->L, c->G, c->src,
                                                                   c->S, nxt, c->ctl.p, c->cnt.p, qk(knxt));
                EMC_CHECK_LAUNCH(c);
            }
            EMC_TRY_CUDA(cudaEventRecord(c->ev[3], st));
            k_collision<<<grid_for(nL, BLK, maxb), BLK, 0, st>>>(c->qc.p, &c->ctl.p->nC, bp, c->L, c->G, c->src,
                                                                c->S, lg, sv, c->bins.p, nxt, c->ctl.p, c->cnt.p,
                                                                qk(knxt));
            EMC_CHECK_LAUNCH(c);
            EMC_TRY_CUDA(cudaEventRecord(c->ev[4], st));
            EMC_TRY_CUDA(cudaMemcpyAsync(c->ctl_host, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
            EMC_TRY_CUDA(cudaStreamSynchronize(st));
            cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]); tm[3] += ms * 1e-3;
            cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]); tm[0] += ms * 1e-3;
            if (c->trace) {       // + the iteration's nuclide-lookups (lookup_counters.py matches ncu launches)
                unsigned long long nlc = 0;
                cudaMemcpy(&nlc, c->cnt.p + CNT_NUCLIDE_LOOKUPS, sizeof(nlc), cudaMemcpyDeviceToHost);
                std::fprintf(stderr, "emc-trace iter %lld nL %lld lookup_ms %.4f sorted %d nl_cum %llu\n",
                             (long long)iterations, (long long)nL, ms, (int)do_sort, nlc);
            }
            cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]); tm[1] += ms * 1e-3;
            cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]); tm[2] += ms * 1e-3;
            int64_t nC = c->ctl_host->nC;
            host_cnt[CNT_EV_LOOKUP] += nL; host_cnt[CNT_EV_ADVANCE] += nL; host_cnt[CNT_EV_COLLISION] += nC;
            host_cnt[CNT_INV_LOOKUP] += 1; host_cnt[CNT_INV_ADVANCE] += 1; host_cnt[CNT_INV_COLLISION] += nC > 0;
            host_cnt[CNT_MAX_INFLIGHT] = std::max(host_cnt[CNT_MAX_INFLIGHT], nL);
            nL = c->ctl_host->nL2;
            std::swap(cur, nxt);
            std::swap(kcur, knxt);
            iterations++;
        }
    }

    // gather results
    unsigned long long dcnt[EMC_N_COUNTERS];
    EMC_TRY_CUDA(cudaMemcpyAsync(dcnt, c->cnt.p, sizeof(dcnt), cudaMemcpyDeviceToHost, st));
    EMC_TRY_CUDA(cudaMemcpyAsync(c->ctl_host, c->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    const Ctl& h = *c->ctl_host;
    for (int k = 0; k < EMC_N_COUNTERS; ++k) res->counters[k] = (int64_t)dcnt[k] + host_cnt[k];
    if (cf.history) {
        res->counters[CNT_INV_LOOKUP] = res->counters[CNT_EV_LOOKUP];
        res->counters[CNT_INV_ADVANCE] = res->counters[CNT_EV_ADVANCE];
        res->counters[CNT_INV_COLLISION] = res->counters[CNT_EV_COLLISION];
    }
    res->counters[CNT_LOG_N] = (int64_t)h.log_n;
    res->counters[CNT_SITE_N] = (int64_t)h.site_n;
    res->counters[CNT_OVF] = h.ovf;
    res->counters[CNT_ERR] = h.err;
    res->counters[CNT_ERR_AUX] = h.err_aux;
    for (int k = 0; k < 4; ++k) res->timings[k] = tm[k];
    res->n_sites = (int64_t)h.site_n;
    res->n_logs = (int64_t)h.log_n;
    res->iterations = iterations;
    res->error = h.err;
    res->error_gid = h.err_aux;
    return 0;
}

extern "C" int emc_run_batch(emc_ctx* c, const emc_batch_args* a, emc_batch_result* res)
{
    if (!c || !a || !res) return fail_arg("emc_run_batch: null argument");
    if (!c->configured) return fail_arg("emc_configure first");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    std::memset(res, 0, sizeof(*res));
    c->G.guard = c->cfg.box_guard ? 1 : 0;      // box guard extension (emc.h), per run
    int64_t l0 = c->launches;
    int reruns = 0;
    if (int rc = presize_logs(c)) return rc;
    for (;;) {
        int rc = run_batch_once(c, a, res);
        if (rc) return rc;
        if (res->error) break;
        int ovf = (int)res->counters[CNT_OVF];
        if (ovf == 0) break;
        // grow-and-rerun (R:107-111, R:122-142): a batch is a pure function of
        // its inputs, so the rerun reproduces the same physics
        size_t need;
        if (ovf == 2) {
            need = std::max<size_t>(2 * c->sites.parent.n, (size_t)res->n_sites + 1024);
            c->sites.release(); c->banks[1 - c->cur_bank].release();
            c->bkey_in.release(); c->bkey_out.release(); c->bidx_in.release(); c->bidx_out.release();
            if ((rc = alloc_sites(c, need))) return rc;
        } else {
            need = std::max<size_t>(2 * c->lg_gid.n, (size_t)res->n_logs + 1024);
            c->lg_gid.release(); c->lg_ord.release(); c->lg_bin.release(); c->lg_val.release();
            c->lkey_in.release(); c->lkey_out.release(); c->lval_out.release();
            if ((rc = alloc_logs(c, need))) return rc;
        }
        reruns++;
    }
    res->reruns = reruns;
    if (res->error) { res->launches = c->launches - l0; return 0; }
    // capacity the next batch's contribution log needs: an unscored batch logs
    // only the k bin, a scored one up to 5 entries per advance event more
    // (K:617-640); grown after this batch's fold (emc_reduce_bins) or at the
    // next batch's start, so the first scoring batch does not overflow and rerun
    if (c->cfg.use_logs) {
        const double est = (double)res->n_logs + (a->score ? 0.0 : 5.0 * (double)res->counters[CNT_EV_ADVANCE]);
        c->log_want = (size_t)(1.25 * est) + 4096;
    }

    // canonical bank: sort this rank's sites by (parent, ordinal)  (R:221-228)
    cudaStream_t st = c->stream;
    int64_t n = res->n_sites;
    if (c->trace) EMC_TRY_CUDA(cudaEventRecord(c->ev[7], st));
    if (n > 0) {
        DSites sv = c->sites.view();
        // site ordinals are < floor(nu/k_run + u) + 1 <= nu_max/k_run + 2: when
        // (parent, ordinal) fits 32 bits, sort 32-bit keys (fewer, narrower passes)
        const double kr = a->k_run > 0.0 ? a->k_run : 1.0;
        const double omax = std::floor(c->nu_max / kr) + 2.0;
        const int ob = omax < 1048576.0 ? bits_for((int64_t)omax) : 20;
        const int pb = bits_for(c->cfg.n_assigned);
        int rc;
        if (pb + ob <= 32) {
            // the 64-bit key buffer (site capacity) holds both 32-bit key arrays
            uint32_t* k32 = reinterpret_cast<uint32_t*>(c->bkey_in.p);
            uint32_t* k32o = k32 + c->bkey_in.n;
            k_bank_keys32<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(sv.parent, sv.ord, n, c->cfg.gid_lo, ob, k32,
                                                                     c->bidx_in.p);
            EMC_CHECK_LAUNCH(c);
            rc = sort_cub(c, k32, k32o, c->bidx_in.p, c->bidx_out.p, (int)n, pb + ob);
        } else {
            k_bank_keys<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(sv.parent, sv.ord, n, c->cfg.gid_lo, c->bkey_in.p,
                                                                   c->bidx_in.p);
            EMC_CHECK_LAUNCH(c);
            rc = sort_cub64(c, c->bkey_in.p, c->bkey_out.p, c->bidx_in.p, c->bidx_out.p, n, pb + 20);
        }
        if (rc) return rc;
        SiteBufs& out = c->banks[1 - c->cur_bank];
        if (out.parent.n < (size_t)n && out.alloc(std::max<size_t>(n, c->sites.parent.n))) return EMC_E_OOM;
        k_bank_gather<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(c->bidx_out.p, n, sv, out.view());
        EMC_CHECK_LAUNCH(c);
    }
    if (c->trace) {
        EMC_TRY_CUDA(cudaEventRecord(c->ev[8], st));
        EMC_TRY_CUDA(cudaEventSynchronize(c->ev[8]));
        float bm = 0;
        cudaEventElapsedTime(&bm, c->ev[7], c->ev[8]);
        std::fprintf(stderr, "emc-trace bank_ms %.4f sites %lld\n", bm, (long long)n);
    }
    c->cur_bank = 1 - c->cur_bank;
    c->bank_n = n;
    // deterministic mode: sort the log by (bin, gid, ordinal) now
    c->log_n = res->n_logs;
    c->lkey_sorted = c->lkey_out.p;
    c->lval_sorted = c->lval_out.p;
    if (c->cfg.use_logs && c->log_n > 0) {
        k_log_keys<<<grid_for(c->log_n, 256, 1 << 30), 256, 0, st>>>(c->lg_gid.p, c->lg_ord.p, c->lg_bin.p,
                                                                     c->log_n, c->cfg.gid_lo, c->gid_bits,
                                                                     c->lkey_in.p);
        EMC_CHECK_LAUNCH(c);
        int bb = bits_for(c->n_bins);
        {
            cub::DoubleBuffer<uint64_t> dk(c->lkey_in.p, c->lkey_out.p);
            cub::DoubleBuffer<double> dv(c->lg_val.p, c->lval_out.p);
            size_t need = 0;
            const int end_bit = bb + c->gid_bits + 17;
            cub::DeviceRadixSort::SortPairs(nullptr, need, dk, dv, (int64_t)c->log_n, 0, end_bit, st);
            if (need > c->cub_tmp.n && c->cub_tmp.alloc(need)) return EMC_E_OOM;
            EMC_TRY_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, need, dk, dv, (int64_t)c->log_n, 0, end_bit,
                                                         st));
            c->launches += (end_bit + 7) / 8;
            c->lkey_sorted = dk.Current();
            c->lval_sorted = dv.Current();
        }
    }
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    res->launches = c->launches - l0;
    return 0;
}

extern "C" int emc_reduce_bins(emc_ctx* c, const double* init, double* out, int64_t n_bins)
{
    if (!c || !out || n_bins != c->n_bins) return fail_arg("emc_reduce_bins: bad arguments");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    if (init) EMC_TRY_CUDA(cudaMemcpyAsync(c->bins_init.p, init, n_bins * 8, cudaMemcpyHostToDevice, st));
    else EMC_TRY_CUDA(cudaMemsetAsync(c->bins_init.p, 0, n_bins * 8, st));
    if (c->cfg.use_logs) {
        if (c->trace) EMC_TRY_CUDA(cudaEventRecord(c->ev[7], st));
        k_log_fold<<<(unsigned)n_bins, LF_THREADS, 0, st>>>(c->lkey_sorted, c->lval_sorted, c->log_n,
                                                                    c->gid_bits + 17, (int32_t)n_bins,
                                                                    c->bins_init.p, c->bins_out.p);
        EMC_CHECK_LAUNCH(c);
        if (c->trace) EMC_TRY_CUDA(cudaEventRecord(c->ev[8], st));
        EMC_TRY_CUDA(cudaMemcpyAsync(out, c->bins_out.p, n_bins * 8, cudaMemcpyDeviceToHost, st));
        EMC_TRY_CUDA(cudaStreamSynchronize(st));
        if (int rc = presize_logs(c)) return rc;   // this batch's log is folded: grow for the next
        if (c->trace) {
            float fm = 0;
            cudaEventElapsedTime(&fm, c->ev[7], c->ev[8]);
            std::fprintf(stderr, "emc-trace fold_ms %.4f logs %lld bins %lld\n", fm, (long long)c->log_n,
                         (long long)n_bins);
        }
    } else {
        std::vector<double> b(n_bins);
        EMC_TRY_CUDA(cudaMemcpyAsync(b.data(), c->bins.p, n_bins * 8, cudaMemcpyDeviceToHost, st));
        EMC_TRY_CUDA(cudaStreamSynchronize(st));
        for (int64_t k = 0; k < n_bins; ++k) out[k] = (init ? init[k] : 0.0) + b[k];
    }
    return 0;
}

extern "C" int emc_bank_size(emc_ctx* c, int64_t* n)
{
    if (!c || !n) return fail_arg("null");
    *n = c->bank_n;
    return 0;
}

extern "C" int emc_bank_device(emc_ctx* c, void* ptrs[9])
{
    if (!c || !ptrs) return fail_arg("null");
    SiteBufs& b = c->bank();
    void* p[9] = {b.parent.p, b.ord.p, b.x.p, b.y.p, b.z.p, b.dx.p, b.dy.p, b.dz.p, b.E.p};
    for (int k = 0; k < 9; ++k) ptrs[k] = p[k];
    return 0;
}

extern "C" int emc_bank_copy(emc_ctx* c, int64_t start, int64_t n, int64_t* parent, int32_t* ord, double* x,
                             double* y, double* z, double* dx, double* dy, double* dz, double* E)
{
    if (!c || start < 0 || n < 0 || start + n > c->bank_n) return fail_arg("emc_bank_copy: range");
    if (n == 0) return 0;
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    SiteBufs& b = c->bank();
    EMC_TRY_CUDA(cudaMemcpyAsync(parent, b.parent.p + start, n * 8, cudaMemcpyDeviceToHost, st));
    EMC_TRY_CUDA(cudaMemcpyAsync(ord, b.ord.p + start, n * 4, cudaMemcpyDeviceToHost, st));
    double* dst[7] = {x, y, z, dx, dy, dz, E};
    double* srcs[7] = {b.x.p, b.y.p, b.z.p, b.dx.p, b.dy.p, b.dz.p, b.E.p};
    for (int k = 0; k < 7; ++k)
        EMC_TRY_CUDA(cudaMemcpyAsync(dst[k], srcs[k] + start, n * 8, cudaMemcpyDeviceToHost, st));
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    return 0;
}

// ------------------------------------------------------------- API ops ---

namespace {
template <class T>
int to_dev(DBuf<T>& b, const T* h, int64_t n, cudaStream_t st)
{
    if (b.alloc(std::max<int64_t>(n, 1))) return EMC_E_OOM;
    if (n) EMC_TRY_CUDA(cudaMemcpyAsync(b.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
    return 0;
}
template <class T>
int to_host(T* h, const DBuf<T>& b, int64_t n, cudaStream_t st)
{
    if (n) EMC_TRY_CUDA(cudaMemcpyAsync(h, b.p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    return 0;
}
}  // namespace

extern "C" int emc_upload_union(emc_ctx* c, const double* ugrid, int64_t n, const int32_t* map,
                                const double* merged)
{
    if (!c || !c->have_lib) return fail_arg("upload a library first");
    if (!ugrid || !map || n < 1) return fail_arg("emc_upload_union: bad arguments");
    const int64_t nn = c->n_nuc;
    for (int64_t i = 1; i < n; ++i)
        if (!(ugrid[i - 1] < ugrid[i])) return fail_arg("union grid must be strictly ascending");
    if (n * nn > ((int64_t)1 << 40)) { g_err = "union index too large"; return EMC_E_RANGE; }
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    // log-hash of the union grid with the library's integer bin map (exact
    // lower bounds of searchsorted(right) - 1, as for the nuclide grids)
    const int64_t nbins = c->L.nbins;
    std::vector<int32_t> hh(nbins);
    int64_t j = 0;
    for (int64_t b = 0; b < nbins; ++b) {
        uint64_t eb = (uint64_t)(c->L.key_lo + b) << c->L.shift;
        double edge;
        std::memcpy(&edge, &eb, 8);
        while (j < n && ugrid[j] <= edge) ++j;
        int64_t start = b == 0 ? 0 : std::max<int64_t>(0, j - 1);
        hh[b] = (int32_t)std::min<int64_t>(start, std::max<int64_t>(0, n - 2));
    }
    c->u_grid.release(); c->u_merged.release(); c->u_hash.release(); c->u_map.release();
    if (c->u_grid.alloc(n) || c->u_hash.alloc(nbins) || c->u_map.alloc(n * nn) ||
        (merged && c->u_merged.alloc(n * nn * 8)))
        return EMC_E_OOM;
    EMC_TRY_CUDA(cudaMemcpy(c->u_grid.p, ugrid, n * sizeof(double), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->u_hash.p, hh.data(), nbins * sizeof(int32_t), cudaMemcpyHostToDevice));
    EMC_TRY_CUDA(cudaMemcpy(c->u_map.p, map, n * nn * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (merged) EMC_TRY_CUDA(cudaMemcpy(c->u_merged.p, merged, n * nn * 8 * sizeof(double), cudaMemcpyHostToDevice));
    c->U = DUnion{c->u_grid.p, c->u_hash.p, c->u_map.p, merged ? c->u_merged.p : nullptr, n, (int32_t)nn, 0};
    return 0;
}

extern "C" int emc_set_accel(emc_ctx* c, int32_t accel)
{
    if (!c) return fail_arg("emc_set_accel: no context");
    if (accel < 0 || accel > 2) return fail_arg("accel must be 0 (binary), 1 (double_index) or 2 (unionized)");
    if (accel >= 1 && !c->U.ugrid) return fail_arg("accel needs a union index (emc_upload_union)");
    if (accel == 2 && !c->U.merged) return fail_arg("accel = unionized needs merged channels");
    c->U.accel = accel;
    return 0;
}

extern "C" int emc_xs_lookup(emc_ctx* c, int64_t n, const int32_t* mats, const double* E, double* sums,
                             double* partials, int32_t max_comp)
{
    if (!c || !c->have_lib) return fail_arg("upload a library first");
    if (n < 0 || (partials && max_comp < c->max_comp)) return fail_arg("emc_xs_lookup: bad arguments");
    for (int64_t i = 0; i < n; ++i)
        if (mats[i] < 0 || mats[i] >= c->n_materials) return fail_arg("unknown material");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<int32_t> dm; DBuf<double> de, ds, dp;
    int rc = to_dev(dm, mats, n, st) | to_dev(de, E, n, st);
    if (rc || ds.alloc(std::max<int64_t>(1, n * 5))) return EMC_E_OOM;
    if (partials && dp.alloc(std::max<int64_t>(1, n * max_comp * 4))) return EMC_E_OOM;
    if (partials) EMC_TRY_CUDA(cudaMemsetAsync(dp.p, 0, n * max_comp * 4 * 8, st));
    if (n) {
        if (c->U.accel == 2)
            k_api_macro<2><<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->L, c->U, n, dm.p, de.p, max_comp, ds.p,
                                                                      partials ? dp.p : nullptr);
        else if (c->U.accel == 1)
            k_api_macro<1><<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->L, c->U, n, dm.p, de.p, max_comp, ds.p,
                                                                      partials ? dp.p : nullptr);
        else
            k_api_macro<0><<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->L, c->U, n, dm.p, de.p, max_comp, ds.p,
                                                                      partials ? dp.p : nullptr);
        EMC_CHECK_LAUNCH(c);
    }
    to_host(sums, ds, n * 5, st);
    if (partials) to_host(partials, dp, n * max_comp * 4, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    dm.release(); de.release(); ds.release(); dp.release();
    return 0;
}

extern "C" int emc_grid_index(emc_ctx* c, int64_t n, const int32_t* entry, const double* E, int32_t* out)
{
    if (!c || !c->have_lib) return fail_arg("upload a library first");
    if (n < 0) return fail_arg("emc_grid_index: bad arguments");
    for (int64_t i = 0; i < n; ++i)
        if (entry[i] < 0 || entry[i] >= c->n_entries) return fail_arg("unknown composition entry");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<int32_t> dk, dout; DBuf<double> de;
    if (to_dev(dk, entry, n, st) || to_dev(de, E, n, st) || dout.alloc(std::max<int64_t>(1, 2 * n))) return EMC_E_OOM;
    if (n) {
        k_api_bracket<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->L, n, dk.p, de.p, dout.p);
        EMC_CHECK_LAUNCH(c);
    }
    to_host(out, dout, 2 * n, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    dk.release(); de.release(); dout.release();
    return 0;
}

extern "C" int emc_locate(emc_ctx* c, int64_t n, const double* pos, int32_t* out)
{
    if (!c || !c->have_geom) return fail_arg("upload a geometry first");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<double> dp; DBuf<int32_t> dout;
    if (to_dev(dp, pos, 3 * n, st) || dout.alloc(std::max<int64_t>(1, 3 * n))) return EMC_E_OOM;
    if (n) { k_api_locate<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->G, n, dp.p, dout.p); EMC_CHECK_LAUNCH(c); }
    to_host(out, dout, 3 * n, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    dp.release(); dout.release();
    return 0;
}

extern "C" int emc_distance(emc_ctx* c, int64_t n, const double* pos, const double* dir, const int32_t* cell,
                            double* dist, int32_t* surf)
{
    if (!c || !c->have_geom) return fail_arg("upload a geometry first");
    for (int64_t i = 0; i < n; ++i)
        if (cell[2 * i] == KIND_FUEL && (cell[2 * i + 1] < 0 || cell[2 * i + 1] >= c->G.n_axial))
            return fail_arg("fuel cell axial index out of range");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<double> dp, dd, ddist; DBuf<int32_t> dc, ds;
    if (to_dev(dp, pos, 3 * n, st) || to_dev(dd, dir, 3 * n, st) || to_dev(dc, cell, 2 * n, st) ||
        ddist.alloc(std::max<int64_t>(1, n)) || ds.alloc(std::max<int64_t>(1, n)))
        return EMC_E_OOM;
    if (n) {
        k_api_distance<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(c->G, n, dp.p, dd.p, dc.p, ddist.p, ds.p);
        EMC_CHECK_LAUNCH(c);
    }
    to_host(dist, ddist, n, st); to_host(surf, ds, n, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    dp.release(); dd.release(); ddist.release(); dc.release(); ds.release();
    return 0;
}

extern "C" int emc_particle_ops(emc_ctx* c, int64_t n, const uint64_t* states, const double* sigma_t, double* iso,
                                double* dcol, uint64_t* st_iso, uint64_t* st_dcol)
{
    if (!c) return fail_arg("null ctx");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<uint64_t> ds, d1, d2; DBuf<double> dsig, diso, dcl;
    if (to_dev(ds, states, n, st) || to_dev(dsig, sigma_t, n, st) || diso.alloc(std::max<int64_t>(1, 3 * n)) ||
        dcl.alloc(std::max<int64_t>(1, n)) || d1.alloc(std::max<int64_t>(1, n)) || d2.alloc(std::max<int64_t>(1, n)))
        return EMC_E_OOM;
    if (n) {
        k_api_particle_ops<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(n, ds.p, dsig.p, diso.p, dcl.p, d1.p, d2.p);
        EMC_CHECK_LAUNCH(c);
    }
    to_host(iso, diso, 3 * n, st); to_host(dcol, dcl, n, st); to_host(st_iso, d1, n, st); to_host(st_dcol, d2, n, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    ds.release(); d1.release(); d2.release(); dsig.release(); diso.release(); dcl.release();
    return 0;
}

namespace {
__global__ void k_qkeys_energy(const int32_t* q, int64_t n, const double* E, uint64_t* keys)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t b = (uint64_t)__double_as_longlong(E[q[i]]);
    keys[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);   // total order of doubles
}
__global__ void k_qkeys_mat(const int32_t* q, int64_t n, const int32_t* mat, uint32_t* keys)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = (uint32_t)mat[q[i]] ^ 0x80000000u;
}
}  // namespace

extern "C" int emc_sort_queue(emc_ctx* c, int64_t n, const int32_t* q, int64_t n_slots, const int32_t* mat,
                              const double* E, int32_t* out)
{
    if (!c || n < 0) return fail_arg("emc_sort_queue: bad arguments");
    for (int64_t i = 0; i < n; ++i) if (q[i] < 0 || q[i] >= n_slots) return fail_arg("queue entry out of range");
    if (n < 2) { if (n == 1) out[0] = q[0]; return 0; }
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<int32_t> dq, dq2, dm; DBuf<double> de; DBuf<uint64_t> k1, k2; DBuf<uint32_t> m1, m2;
    if (to_dev(dq, q, n, st) || to_dev(dm, mat, n_slots, st) || to_dev(de, E, n_slots, st) || dq2.alloc(n) ||
        k1.alloc(n) || k2.alloc(n) || m1.alloc(n) || m2.alloc(n))
        return EMC_E_OOM;
    // two stable passes == the reference's argsort(E) then argsort(mat) (K:1026-1033)
    k_qkeys_energy<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(dq.p, n, de.p, k1.p);
    EMC_CHECK_LAUNCH(c);
    int rc = sort_cub64(c, k1.p, k2.p, dq.p, dq2.p, n, 64);
    if (rc) return rc;
    k_qkeys_mat<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(dq2.p, n, dm.p, m1.p);
    EMC_CHECK_LAUNCH(c);
    rc = sort_cub64(c, m1.p, m2.p, dq2.p, dq.p, n, 32);
    if (rc) return rc;
    to_host(out, dq, n, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    dq.release(); dq2.release(); dm.release(); de.release(); k1.release(); k2.release(); m1.release(); m2.release();
    return 0;
}

extern "C" int emc_replay_bins(emc_ctx* c, int64_t n, const int32_t* bin, const double* val, int32_t n_bins,
                               double* sums)
{
    if (!c || n < 0 || n_bins < 1) return fail_arg("emc_replay_bins: bad arguments");
    for (int64_t i = 0; i < n; ++i) if (bin[i] < 0 || bin[i] >= n_bins) return fail_arg("bin out of range");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    int pb = bits_for(n), bb = bits_for(n_bins);
    if (pb + bb > 64) { g_err = "replay too large"; return EMC_E_RANGE; }
    DBuf<int32_t> db; DBuf<double> dv, dv2, dinit, dout; DBuf<uint64_t> k1, k2;
    if (to_dev(db, bin, n, st) || to_dev(dv, val, n, st) || dv2.alloc(std::max<int64_t>(n, 1)) ||
        k1.alloc(std::max<int64_t>(n, 1)) || k2.alloc(std::max<int64_t>(n, 1)) || dinit.alloc(n_bins) ||
        dout.alloc(n_bins))
        return EMC_E_OOM;
    EMC_TRY_CUDA(cudaMemsetAsync(dinit.p, 0, n_bins * 8, st));
    if (n) {
        k_replay_keys<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(db.p, n, pb, k1.p);
        EMC_CHECK_LAUNCH(c);
        int rc = sort_cub64(c, k1.p, k2.p, dv.p, dv2.p, n, pb + bb);
        if (rc) return rc;
    }
    if (n_bins > 0) {
        k_log_fold<<<(unsigned)n_bins, LF_THREADS, 0, st>>>(k2.p, dv2.p, n, pb, n_bins, dinit.p, dout.p);
        EMC_CHECK_LAUNCH(c);
    }
    to_host(sums, dout, n_bins, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    db.release(); dv.release(); dv2.release(); k1.release(); k2.release(); dinit.release(); dout.release();
    return 0;
}

extern "C" int emc_lcg_skip(emc_ctx* c, int64_t n, const uint64_t* s, const uint64_t* k, uint64_t* out)
{
    if (!c) return fail_arg("null ctx");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<uint64_t> ds, dk, dout;
    if (to_dev(ds, s, n, st) || to_dev(dk, k, n, st) || dout.alloc(std::max<int64_t>(n, 1))) return EMC_E_OOM;
    if (n) { k_api_lcg_skip<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(n, ds.p, dk.p, dout.p); EMC_CHECK_LAUNCH(c); }
    to_host(out, dout, n, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    ds.release(); dk.release(); dout.release();
    return 0;
}

extern "C" int emc_libm_eval(emc_ctx* c, int64_t n, const double* x, double* out)
{
    if (!c) return fail_arg("null ctx");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<double> dx, dout;
    if (to_dev(dx, x, n, st) || dout.alloc(std::max<int64_t>(3 * n, 1))) return EMC_E_OOM;
    if (n) { k_api_libm<<<grid_for(n, 128, 1 << 30), 128, 0, st>>>(n, dx.p, dout.p); EMC_CHECK_LAUNCH(c); }
    to_host(out, dout, 3 * n, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    dx.release(); dout.release();
    return 0;
}

extern "C" int emc_div_eval(emc_ctx* c, int64_t n, const double* num, const double* den, double* out)
{
    if (!c) return fail_arg("null ctx");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<double> dn, dd, dout;
    if (to_dev(dn, num, n, st) || to_dev(dd, den, n, st) || dout.alloc(std::max<int64_t>(2 * n, 1))) return EMC_E_OOM;
    if (n) { k_api_div<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(n, dn.p, dd.p, dout.p); EMC_CHECK_LAUNCH(c); }
    to_host(out, dout, 2 * n, st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    dn.release(); dd.release(); dout.release();
    return 0;
}

// lookup microbenchmark: the staged path's sort key of each (E, mat) pair
namespace emc {
__global__ void k_bench_keys(int32_t n, DLib L, const double* __restrict__ E, const int32_t* __restrict__ M, QKeys K,
                             int32_t* __restrict__ idx)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { K.keys[i] = lookup_key(L, K, E[i], M[i]); idx[i] = i; }
}

__global__ void k_bench_permute(int32_t n, const int32_t* __restrict__ perm, const double* __restrict__ E,
                                const int32_t* __restrict__ M, double* __restrict__ Eo, int32_t* __restrict__ Mo)
{
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { Eo[i] = E[perm[i]]; Mo[i] = M[perm[i]]; }
}
}  // namespace emc

// test/tuning entry point: time k_lookup_bench<variant> over n (mat, E) pairs
extern "C" int emc_bench_lookup(emc_ctx* c, int64_t n, const int32_t* mats, const double* E, int32_t variant,
                                int32_t iters, double* ms_out, double* checksum)
{
    if (!c || !c->have_lib || n < 1 || iters < 1) return fail_arg("emc_bench_lookup: bad arguments");
    EMC_TRY_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = c->stream;
    DBuf<int32_t> dm; DBuf<double> de, dout;
    if (to_dev(dm, mats, n, st) || to_dev(de, E, n, st) || dout.alloc(n * 17)) return EMC_E_OOM;
    int grid = c->sm_count * 16;
    DBuf<uint32_t> dk;          // variant 9: pairs put in sort-key order, keys kept for the kernel
    if (variant == 9) {
        if (!c->staged || !c->configured) return fail_arg("emc_bench_lookup: variant 9 needs a configured staged library");
        DBuf<uint32_t> k0; DBuf<int32_t> i0, i1, m1; DBuf<double> e1;
        if (dk.alloc(n) || k0.alloc(n) || i0.alloc(n) || i1.alloc(n) || m1.alloc(n) || e1.alloc(n)) return EMC_E_OOM;
        k_bench_keys<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>((int32_t)n, c->L, de.p, dm.p,
            QKeys{k0.p, c->ebin_bits, c->ebin_shift, c->mat_bits, c->band_bits}, i0.p);
        EMC_CHECK_LAUNCH(c);
        if (int rc = sort_cub(c, k0.p, dk.p, i0.p, i1.p, (int)n, c->key_bits)) return rc;
        k_bench_permute<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>((int32_t)n, i1.p, de.p, dm.p, e1.p, m1.p);
        EMC_CHECK_LAUNCH(c);
        EMC_TRY_CUDA(cudaMemcpyAsync(de.p, e1.p, n * 8, cudaMemcpyDeviceToDevice, st));
        EMC_TRY_CUDA(cudaMemcpyAsync(dm.p, m1.p, n * 4, cudaMemcpyDeviceToDevice, st));
        EMC_TRY_CUDA(cudaStreamSynchronize(st));
        k0.release(); i0.release(); i1.release(); m1.release(); e1.release();
    }
    float total = 0;
    for (int it = 0; it <= iters; ++it) {
        EMC_TRY_CUDA(cudaEventRecord(c->ev[0], st));
        if (variant == 8) {
            EMC_TRY_CUDA(lk_launch<1>(c->lk_cfg, c->L, nullptr, n, c->S, 1, c->cnt.p, de.p, dm.p, dout.p, c->sm_count,
                                      c->lk_smem, st));
        } else if (variant == 9) {
            EMC_TRY_CUDA(lk_launch_piped<1>(c->L, nullptr, n, c->S, 1, c->cnt.p, de.p, dm.p, dout.p, c->sm_count,
                                            c->lk_smem, st, nullptr, lk_keys(c, dk.p)));
        } else {
            k_lookup_bench<<<grid, 256, 0, st>>>((int32_t)n, c->L, de.p, dm.p, dout.p);
        }
        EMC_CHECK_LAUNCH(c);
        EMC_TRY_CUDA(cudaEventRecord(c->ev[1], st));
        EMC_TRY_CUDA(cudaEventSynchronize(c->ev[1]));
        float ms;
        cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
        if (it > 0) total += ms;   // first launch = warm-up
    }
    *ms_out = total / iters;
    std::vector<double> h(std::min<int64_t>(n, 1024));
    to_host(h.data(), dout, (int64_t)h.size(), st);
    EMC_TRY_CUDA(cudaStreamSynchronize(st));
    double cs = 0;
    for (double v : h) cs += v;
    *checksum = cs;
    dm.release(); de.release(); dout.release(); dk.release();
    return 0;
}

#include "emc_group.cuh"
