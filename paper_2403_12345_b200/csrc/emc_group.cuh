// Single-process multi-GPU group (SURVEY.md 8b "emc_init(devices[], W)",
// "emc_exchange_bank", "emc_allreduce_bins"): the C-ABI form of what
// replication.py / distributed.py do for the Python host, for a host in any
// language.  Rank r is a context configured for the particle block
// [r*P/W, (r+1)*P/W) (contiguous blocks: the global canonical bank is the
// rank-ordered concatenation of the rank banks, R:221-228).  Per batch, after
// every rank's emc_run_batch:
//   emc_group_reduce_bins  -- tallies: deterministic = chained fold (rank r
//                             starts from rank r-1's sums: bit-identical to one
//                             rank), fast = rank-ordered sum of the rank bins
//   emc_group_exchange_bank -- each rank receives exactly the window of the
//                             global bank its block resamples from (R:271-280,
//                             T:188-200), copied device to device (peer copies
//                             over NVLink), and installs it as its source.
// Included by emc_engine.cu (needs emc_ctx).
#pragma once

struct emc_group {
    std::vector<emc_ctx*> ranks;
    std::vector<SiteBufs> win;          // per rank: its resampling window (x..E used), on its device
};

namespace emc_grp {

// transport.py:188-200 / distributed.resample_index: the bank index particle g
// resamples, with the device's expression (floor(((g + u) * n) / ppb))
inline int64_t resample_index(int64_t g, int64_t n, int64_t ppb, double u)
{
    if (n >= ppb) {
        volatile double t = ((double)g + u) * (double)n;
        int64_t i = (int64_t)std::floor(t / (double)ppb);
        return std::min<int64_t>(std::max<int64_t>(i, 0), n - 1);
    }
    return g % n;
}

// distributed.needed_window: (lo, length) of the cyclic bank window [g_lo, g_hi) resamples from
inline void needed_window(int64_t g_lo, int64_t g_hi, int64_t n, int64_t ppb, double u, int64_t& lo, int64_t& len)
{
    lo = 0; len = 0;
    if (g_hi <= g_lo || n < 1) return;
    if (n >= ppb) {
        const int64_t a = resample_index(g_lo, n, ppb, u), b = resample_index(g_hi - 1, n, ppb, u);
        lo = a; len = b - a + 1;
        return;
    }
    if (g_hi - g_lo >= n) { lo = 0; len = n; return; }
    lo = g_lo % n; len = g_hi - g_lo;
}

}  // namespace emc_grp

extern "C" int emc_group_create(emc_ctx* const* ctxs, int32_t n, emc_group** out)
{
    if (!ctxs || n < 1 || !out) return fail_arg("emc_group_create: bad arguments");
    for (int32_t r = 0; r < n; ++r)
        if (!ctxs[r] || !ctxs[r]->configured) return fail_arg("emc_group_create: every rank must be configured");
    emc_group* g = new emc_group();
    g->ranks.assign(ctxs, ctxs + n);
    g->win.resize(n);
    // peer access between the ranks' devices (NVLink); already-enabled is fine
    for (int32_t a = 0; a < n; ++a)
        for (int32_t b = 0; b < n; ++b) {
            const int da = g->ranks[a]->device, db = g->ranks[b]->device;
            int can = 0;
            if (da == db || cudaDeviceCanAccessPeer(&can, da, db) != cudaSuccess || !can) continue;
            cudaSetDevice(da);
            if (cudaDeviceEnablePeerAccess(db, 0) != cudaSuccess) cudaGetLastError();
        }
    *out = g;
    return 0;
}

extern "C" void emc_group_destroy(emc_group* g)
{
    if (!g) return;
    for (size_t r = 0; r < g->win.size(); ++r) {
        cudaSetDevice(g->ranks[r]->device);
        SiteBufs& w = g->win[r];
        w.parent.release(); w.ord.release(); w.x.release(); w.y.release(); w.z.release();
        w.dx.release(); w.dy.release(); w.dz.release(); w.E.release();
    }
    delete g;
}

extern "C" int emc_group_reduce_bins(emc_group* g, double* out, int64_t n_bins)
{
    if (!g || !out) return fail_arg("emc_group_reduce_bins: bad arguments");
    const size_t W = g->ranks.size();
    std::vector<double> prev(n_bins, 0.0), mine(n_bins, 0.0);
    if (g->ranks[0]->cfg.use_logs) {
        for (size_t r = 0; r < W; ++r) {               // the chain: rank r folds from rank r-1's sums
            if (int rc = emc_reduce_bins(g->ranks[r], r ? prev.data() : nullptr, mine.data(), n_bins)) return rc;
            prev.swap(mine);
        }
    } else {
        for (size_t r = 0; r < W; ++r) {               // rank-ordered left fold (R:238-240)
            if (int rc = emc_reduce_bins(g->ranks[r], nullptr, mine.data(), n_bins)) return rc;
            for (int64_t k = 0; k < n_bins; ++k) prev[k] += mine[k];
        }
    }
    std::memcpy(out, prev.data(), n_bins * sizeof(double));
    return 0;
}

extern "C" int emc_group_exchange_bank(emc_group* g, int64_t ppb, double u, int64_t* out_n)
{
    if (!g || ppb < 1) return fail_arg("emc_group_exchange_bank: bad arguments");
    const int64_t W = (int64_t)g->ranks.size();
    std::vector<int64_t> offs(W + 1, 0);
    for (int64_t r = 0; r < W; ++r) offs[r + 1] = offs[r] + g->ranks[r]->bank_n;
    const int64_t n = offs[W];
    if (out_n) *out_n = n;
    if (n < 1) return fail_arg("no fission sites banked (population collapse)");
    for (int64_t q = 0; q < W; ++q) {
        emc_ctx* dst = g->ranks[q];
        int64_t lo, len;
        emc_grp::needed_window(q * ppb / W, (q + 1) * ppb / W, n, ppb, u, lo, len);
        EMC_TRY_CUDA(cudaSetDevice(dst->device));
        SiteBufs& w = g->win[q];
        if ((int64_t)w.x.n < std::max<int64_t>(len, 1)) {
            w.x.release(); w.y.release(); w.z.release(); w.dx.release(); w.dy.release(); w.dz.release(); w.E.release();
            const size_t cap = (size_t)std::max<int64_t>(len, 1) * 5 / 4 + 1024;
            if (w.x.alloc(cap) || w.y.alloc(cap) || w.z.alloc(cap) || w.dx.alloc(cap) || w.dy.alloc(cap) ||
                w.dz.alloc(cap) || w.E.alloc(cap))
                return EMC_E_OOM;
        }
        double* const wd[7] = {w.x.p, w.y.p, w.z.p, w.dx.p, w.dy.p, w.dz.p, w.E.p};
        // the window in order: up to two linear segments of the cyclic range
        int64_t seg[2][2];
        int nseg = 0;
        if (len > 0) {
            if (lo + len <= n) { seg[0][0] = lo; seg[0][1] = lo + len; nseg = 1; }
            else { seg[0][0] = lo; seg[0][1] = n; seg[1][0] = 0; seg[1][1] = lo + len - n; nseg = 2; }
        }
        int64_t wpos = 0;
        for (int sgi = 0; sgi < nseg; ++sgi) {
            for (int64_t r = 0; r < W; ++r) {          // the pieces of segment sgi owned by rank r
                const int64_t a = std::max(seg[sgi][0], offs[r]), b = std::min(seg[sgi][1], offs[r + 1]);
                if (b <= a) continue;
                emc_ctx* src = g->ranks[r];
                SiteBufs& bk = src->bank();
                const double* const sd[7] = {bk.x.p, bk.y.p, bk.z.p, bk.dx.p, bk.dy.p, bk.dz.p, bk.E.p};
                for (int f = 0; f < 7; ++f)
                    EMC_TRY_CUDA(cudaMemcpyPeerAsync(wd[f] + wpos + (a - seg[sgi][0]), dst->device,
                                                     sd[f] + (a - offs[r]), src->device,
                                                     (size_t)(b - a) * sizeof(double), dst->stream));
            }
            wpos += seg[sgi][1] - seg[sgi][0];
        }
        EMC_TRY_CUDA(cudaStreamSynchronize(dst->stream));
        const void* ptrs[7] = {w.x.p, w.y.p, w.z.p, w.dx.p, w.dy.p, w.dz.p, w.E.p};
        if (int rc = emc_set_source_window(dst, ptrs, n, u, lo)) return rc;
    }
    return 0;
}
