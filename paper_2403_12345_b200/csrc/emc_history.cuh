// History-based executor on the GPU (reference: run_history_batch,
// kernels.py:1043-1089): each thread transports one particle birth to death,
// then claims the next index of the batch.  Same device ops as the event
// kernels (identical arithmetic => identical physics); buffers are appended
// with per-thread atomics because threads diverge freely.  This is the
// paper's "history-based" comparison point, not the fast path.
#pragma once
#include "emc_kernels.cuh"

namespace emc {

// Accumulators of one thread's histories (flushed once per thread).
struct HistAcc {
    unsigned long long ev_l = 0, ev_a = 0, ev_c = 0, interp = 0, interp_score = 0, nuc_lookups = 0;
    unsigned long long captures = 0, fissions = 0, leaks = 0, maxdraws = 0, maxhist = 0;
    int clamps = 0;
};

// Warp-cooperative macro_tcf for ONE particle (all 32 lanes call it with the
// same material and energy): the lanes gather 32 nuclides at a time and every
// lane replays the sequential fold over shuffles (k_lookup_warp<32>'s scheme:
// same operations, same order, bit-identical sums); lane 0 writes the sigma_t
// checkpoints.
__device__ __forceinline__ void macro_tcf_warp32(const DLib& L, int32_t m, double E, double& st, double& sc,
                                                 double& sf, double& snf, double* ck, int32_t nck, int64_t cks)
{
    const int lane = (int)(threadIdx.x & 31u);
    const int32_t grp = __ldg(L.mat_group + m);
    const int32_t e0 = __ldg(L.grp_off + grp), ncomp = __ldg(L.grp_off + grp + 1) - e0;
    const int32_t bin = energy_bin(E, L);
    st = 0.0; sc = 0.0; sf = 0.0; snf = 0.0;
    for (int32_t k0 = 0; k0 < ncomp; k0 += 32) {
        double t = 0.0, cc = 0.0, f = 0.0, den = 0.0, dn = 0.0;
        const int32_t k = k0 + lane;
        if (k < ncomp) {
            const NucRef r = L.gnuc[e0 + k];
            const DD w = L.ddT[(int64_t)k * L.n_mat + m];
            den = w.den; dn = w.dn;
            const Rec* __restrict__ R = L.rec + r.g0;
            const int32_t last = r.glen - 1;
            if (last == 0) {
                const Rec r0 = R[0];
                t = r0.t; cc = r0.c; f = r0.f;
            } else {
                int32_t j = __ldg(L.hash + r.hrow + bin);
                Rec r0 = R[j], r1 = R[j + 1];
                while (r1.E <= E && j + 1 < last) { ++j; r0 = r1; r1 = R[j + 1]; }
                if (j == 0 && E <= r0.E) { t = r0.t; cc = r0.c; f = r0.f; }
                else if (E >= r1.E) { t = r1.t; cc = r1.c; f = r1.f; }
                else {
                    const double fr = frac(E, r0.E, r1.E);
                    t = lerp(r0.t, r1.t, fr);
                    cc = lerp(r0.c, r1.c, fr);
                    f = lerp(r0.f, r1.f, fr);
                }
            }
        }
        const int kn = min(32, ncomp - k0);
        for (int j = 0; j < kn; ++j) {
            const double tj = __shfl_sync(kFull, t, j), cj = __shfl_sync(kFull, cc, j);
            const double fj = __shfl_sync(kFull, f, j), dj = __shfl_sync(kFull, den, j);
            const double dnj = __shfl_sync(kFull, dn, j);
            st = __dadd_rn(st, __dmul_rn(dj, tj));
            sc = __dadd_rn(sc, __dmul_rn(dj, cj));
            sf = __dadd_rn(sf, __dmul_rn(dj, fj));
            snf = __dadd_rn(snf, __dmul_rn(dnj, fj));
            if (ck && lane == 0 && ((k0 + j + 1) & (kCkptStride - 1)) == 0) {
                const int32_t row = (k0 + j + 1) / kCkptStride - 1;
                if (row < nck) ck[(int64_t)row * cks] = st;
            }
        }
    }
    __syncwarp();        // lane 0's checkpoint stores are visible to the whole warp (collision walk)
}

// One particle from "awaiting its cross-section lookup" to death, event after
// event (the loop body of run_history_batch, K:1055-1086, with the event
// kernels' arithmetic).  Returns true when the history failed (error set).
// WARP: the 32 lanes of a warp carry ONE particle -- lookups are
// warp-cooperative (macro_tcf_warp32), everything else runs redundantly on
// identical values in every lane (so control flow stays uniform), and only
// lane 0 touches shared state (atomics, log / bank / tally writes), its
// claimed indices broadcast by shuffles.
template <bool WARP = false>
__device__ __forceinline__ bool transport_to_death(int32_t s, int64_t g, uint64_t& rng, int32_t& draws,
                                                   int32_t& ordc, int32_t& hist, double x, double y, double z,
                                                   double dx, double dy, double dz, double E, int kd, int32_t ax,
                                                   int32_t m, const BatchP& bp, const DLib& L, const DGeom& G,
                                                   const DSlots& S, const DLog& lg, const DSites& sb, double* bins,
                                                   Ctl* ctl, unsigned long long* cnt, const DMesh& M, HistAcc& A)
{
    double* ck = ckpt_of(S, s);
    const bool lead = !WARP || (threadIdx.x & 31u) == 0;
    auto claim = [&](unsigned long long* ctr, unsigned long long k) -> unsigned long long {
        unsigned long long at = 0;
        if (lead) at = atomicAdd(ctr, k);
        if (WARP) at = __shfl_sync(kFull, at, 0);
        return at;
    };
    for (;;) {
        // --- lookup (K:573-710)
        double st, sc, sf, snf;
        if (WARP) macro_tcf_warp32(L, m, E, st, sc, sf, snf, bp.fused ? ck : nullptr, S.nck, S.ck_row);
        else macro_tcf(L, m, E, st, sc, sf, snf, bp.fused ? ck : nullptr, S.nck, S.ck_row);
        A.interp += 4ull * (unsigned long long)(L.mat_off[m + 1] - L.mat_off[m]);
        A.nuc_lookups += (unsigned long long)(L.mat_off[m + 1] - L.mat_off[m]);
        A.ev_l += 1;
        // --- advance (K:713-811)
        A.ev_a += 1;
        if (!(st > 0.0)) { if (lead) set_error(ctl, cnt, ERR_NONPOSITIVE_SIGMA, g); return true; }
        double u = draw(rng, draws);
        double d_coll = __ddiv_rn(-emc_log(__dsub_rn(1.0, u)), st);
        int32_t surf;
        double dist = boundary_distance(x, y, z, dx, dy, dz, kd, ax, G, surf);
        if (surf < 0) { if (lead) set_error(ctl, cnt, ERR_NO_SURFACE, g); return true; }
        bool crossing = !(d_coll < dist);
        double ell = crossing ? dist : d_coll;
        if (bp.score) {
            int32_t base = (kd == KIND_FUEL ? ax : G.n_axial) * 5;
            double fl = __dmul_rn(1.0, ell), v[5];
            if (bp.fused) {
                v[1] = __dmul_rn(fl, st); v[2] = __dmul_rn(fl, __dadd_rn(sc, sf));
                v[3] = __dmul_rn(fl, sf); v[4] = __dmul_rn(fl, snf);
            } else {
                double st2, sc2, sf2, snf2;
                macro_tcf_simple(L, m, E, st2, sc2, sf2, snf2, nullptr, 0);
                A.interp_score += 3ull * (unsigned long long)(L.mat_off[m + 1] - L.mat_off[m]);
                v[1] = __dmul_rn(fl, st2); v[2] = __dmul_rn(fl, __dadd_rn(sc2, sf2));
                v[3] = __dmul_rn(fl, sf2); v[4] = __dmul_rn(fl, snf2);
            }
            v[0] = fl;
            for (int k = 0; k < 5; ++k) {
                if (v[k] == 0.0) continue;
                if (bp.use_logs) {
                    unsigned long long at = claim(&ctl->log_n, 1ULL);
                    if (!lead) {}
                    else if (at >= (unsigned long long)lg.cap) atomicExch(&ctl->ovf, 1);
                    else { lg.gid[at] = g; lg.ord[at] = ordc; lg.bin[at] = base + k; lg.val[at] = v[k]; }
                    ordc += 1; hist += 1;
                } else {
                    if (lead) atomicAdd(bins + base + k, v[k]);
                }
            }
            if (hist > kMaxHistLog) { if (lead) set_error(ctl, cnt, ERR_RUNAWAY_HISTORY, g); return true; }
            if (M.on && lead) score_mesh(M, x, y, z, dx, dy, dz, ell, st);
        }
        x = __dadd_rn(x, __dmul_rn(dx, ell));
        y = __dadd_rn(y, __dmul_rn(dy, ell));
        z = __dadd_rn(z, __dmul_rn(dz, ell));
        bool died = false, guarded = false;
        if (!crossing && G.guard && box_guard(x, y, z, dx, dy, dz, G)) {   // box guard (extension)
            if (lead) atomicAdd(cnt + CNT_BOX_GUARD, 1ull);
            guarded = true;
            if (G.vacuum) { A.leaks += 1; died = true; }
            else kd = locate_point(x, y, z, G, ax, m);
        }
        if (guarded) {
        } else if (crossing && G.vacuum && surf >= SURF_XMIN && surf <= SURF_ZMAX) {
            A.leaks += 1; died = true;                 // vacuum boundary (extension)
        } else if (crossing) {
            if (surf >= SURF_XMIN && surf <= SURF_ZMAX) {
                if (surf == SURF_XMIN || surf == SURF_XMAX) dx = -dx;
                else if (surf == SURF_YMIN || surf == SURF_YMAX) dy = -dy;
                else dz = -dz;
            }
            x = __dadd_rn(x, __dmul_rn(dx, kNudge));
            y = __dadd_rn(y, __dmul_rn(dy, kNudge));
            z = __dadd_rn(z, __dmul_rn(dz, kNudge));
            if (surf == SURF_CYL) {
                if (kd == KIND_FUEL) { kd = KIND_MOD; ax = -1; }
                else { kd = KIND_FUEL; ax = axial_index(z, G.n_axial, G.height); }
            } else if (surf >= SURF_AXIAL_BASE && surf < SURF_LATTICE) {
                int32_t jpl = surf - SURF_AXIAL_BASE;
                ax = dz > 0.0 ? jpl : jpl - 1;
            }
            m = kd == KIND_FUEL ? G.fuel_mats[ax] : G.mod_mat;
            if (G.guard && box_guard(x, y, z, dx, dy, dz, G)) {
                if (lead) atomicAdd(cnt + CNT_BOX_GUARD, 1ull);
                if (G.vacuum) { A.leaks += 1; died = true; }
                else kd = locate_point(x, y, z, G, ax, m);
            }
        } else {
            // --- collision (K:814-923)
            A.ev_c += 1;
            double kval = __dmul_rn(1.0, __ddiv_rn(snf, st));
            if (bp.use_logs) {
                if (kval != 0.0) {
                    unsigned long long at = claim(&ctl->log_n, 1ULL);
                    if (!lead) {}
                    else if (at >= (unsigned long long)lg.cap) atomicExch(&ctl->ovf, 1);
                    else { lg.gid[at] = g; lg.ord[at] = ordc; lg.bin[at] = bp.kbin; lg.val[at] = kval; }
                    ordc += 1; hist += 1;
                    if (hist > kMaxHistLog) { if (lead) set_error(ctl, cnt, ERR_RUNAWAY_HISTORY, g); return true; }
                }
            } else {
                if (lead) atomicAdd(bins + bp.kbin, kval);
            }
            int32_t e0 = L.mat_off[m], e1 = L.mat_off[m + 1];
            int32_t bin = energy_bin(E, L);
            double u1 = draw(rng, draws);
            double tgt = __dmul_rn(u1, st);
            double pt_sel;
            int32_t ksel = select_nuclide(L, ck, S.nck, S.ck_row, e0, e1, bin, E, u1, tgt, bp.fused != 0, pt_sel, A.interp);
            const Comp cs = load_comp(L.comp + ksel);
            double s_s, s_c, s_f;
            micro_scf(L, cs, bin, E, s_s, s_c, s_f);
            A.interp += 3;
            double ps = __dmul_rn(cs.den, s_s), pc = __dmul_rn(cs.den, s_c);
            double u2 = draw(rng, draws);
            double tgt2 = __dmul_rn(u2, pt_sel);
            if (tgt2 < ps) {
                double u3 = draw(rng, draws), u4 = draw(rng, draws);
                isotropic(u3, u4, dx, dy, dz);
                double u5 = draw(rng, draws);
                double ep = __dmul_rn(E, __dadd_rn(bp.alpha, __dmul_rn(__dsub_rn(1.0, bp.alpha), u5)));
                E = clamp_energy(ep, L, A.clamps);
            } else if (tgt2 < __dadd_rn(ps, pc)) {
                A.captures += 1; died = true;
            } else {
                A.fissions += 1; died = true;
                double u5 = draw(rng, draws);
                int64_t ns = (int64_t)floor(__dadd_rn(__ddiv_rn(__ldg(L.nu + cs.nid), bp.k_run), u5));
                if (ns > 0) {
                    unsigned long long at = claim(&ctl->site_n, (unsigned long long)ns);
                    for (int64_t ms = 0; ms < ns; ++ms) {
                        double ua = draw(rng, draws), ub = draw(rng, draws), sx, sy, sz;
                        isotropic(ua, ub, sx, sy, sz);
                        double uc = draw(rng, draws);
                        double es = clamp_energy(__dmul_rn(-bp.fission_t, emc_log(__dsub_rn(1.0, uc))), L, A.clamps);
                        unsigned long long w = at + ms;
                        if (!lead) continue;
                        if (w >= (unsigned long long)sb.cap) { atomicExch(&ctl->ovf, 2); continue; }
                        sb.parent[w] = g; sb.ord[w] = (int32_t)ms;
                        sb.x[w] = x; sb.y[w] = y; sb.z[w] = z;
                        sb.dx[w] = sx; sb.dy[w] = sy; sb.dz[w] = sz; sb.E[w] = es;
                    }
                }
            }
        }
        if (draws >= kStride) { if (lead) set_error(ctl, cnt, ERR_STREAM_OVERLAP, g); return true; }
        if (died) break;
    }
    return false;
}

__device__ __forceinline__ void flush_hist_acc(const HistAcc& A, unsigned long long sourced, unsigned long long* cnt)
{
    if (A.ev_l) atomicAdd(cnt + CNT_EV_LOOKUP, A.ev_l);
    if (A.ev_a) atomicAdd(cnt + CNT_EV_ADVANCE, A.ev_a);
    if (A.ev_c) atomicAdd(cnt + CNT_EV_COLLISION, A.ev_c);
    if (A.interp) atomicAdd(cnt + CNT_INTERP_TRANSPORT, A.interp);
    if (A.nuc_lookups) atomicAdd(cnt + CNT_NUCLIDE_LOOKUPS, A.nuc_lookups);
    if (A.interp_score) atomicAdd(cnt + CNT_INTERP_SCORE, A.interp_score);
    if (A.captures) atomicAdd(cnt + CNT_CAPTURES, A.captures);
    if (A.fissions) atomicAdd(cnt + CNT_FISSIONS, A.fissions);
    if (A.leaks) atomicAdd(cnt + CNT_LEAKS, A.leaks);
    if (sourced) atomicAdd(cnt + CNT_SOURCED, sourced);
    if (A.clamps) atomicAdd(cnt + CNT_CLAMPS, (unsigned long long)A.clamps);
    if (A.maxdraws) atomicMax(cnt + CNT_MAX_DRAWS, A.maxdraws);
    if (A.maxhist) atomicMax(cnt + CNT_MAX_HIST_LOG, A.maxhist);
}

__global__ void __launch_bounds__(128) k_history(BatchP bp, DLib L, DGeom G, DSrc src, DSlots S, DLog lg,
                                                 DSites sb, double* bins, Ctl* ctl, unsigned long long* cnt,
                                                 int64_t nthreads, DMesh M)
{
    const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= nthreads) return;
    HistAcc A;
    unsigned long long sourced = 0;
    const int32_t s = (int32_t)slot;
    for (;;) {
        if (*(volatile int32_t*)&ctl->err) break;
        unsigned long long idx = atomicAdd(&ctl->cursor, 1ULL);
        if (idx >= (unsigned long long)bp.n_assigned) break;
        int64_t g = bp.g_lo + (int64_t)idx;
        sourced += 1;
        if (!source_particle(s, g, bp, L, G, src, S, ctl, A.clamps)) break;
        const PState& p0 = S.ps[s];
        uint64_t rng = p0.b.rng;
        int32_t draws = p0.d.draws, ordc = 0, hist = 0;
        if (transport_to_death(s, g, rng, draws, ordc, hist, p0.a.x, p0.a.y, p0.a.z, p0.b.dx, p0.b.dy, p0.b.dz,
                               p0.a.E, p0.d.kind, p0.d.axial, p0.d.mat, bp, L, G, S, lg, sb, bins, ctl, cnt, M, A))
            break;
        A.maxdraws = max(A.maxdraws, (unsigned long long)draws);
        A.maxhist = max(A.maxhist, (unsigned long long)hist);
    }
    flush_hist_acc(A, sourced, cnt);
}

// Event-mode small-population finish: every particle of the lookup queue
// (state in its PState line, exactly as the event kernels left it) is carried
// to death by one thread, history-style.  Physics is schedule-invariant
// (acceptance criterion 1): the same events happen with the same arithmetic
// and draws, only no longer in lock-step sweeps -- a few thousand in-flight
// particles no longer pay a chain of launch-latency-bound sweeps each.
__global__ void __launch_bounds__(128) k_finish(const int32_t* __restrict__ q, int64_t n, BatchP bp, DLib L,
                                                DGeom G, DSlots S, DLog lg, DSites sb, double* bins, Ctl* ctl,
                                                unsigned long long* cnt, DMesh M)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    HistAcc A;
    const int32_t s = q[i];
    const PState p = S.ps[s];
    if (!*(volatile int32_t*)&ctl->err) {
        uint64_t rng = p.b.rng;
        int32_t draws = p.d.draws, ordc = p.d.ordctr, hist = p.d.histlog;
        if (!transport_to_death(s, p.d.gid, rng, draws, ordc, hist, p.a.x, p.a.y, p.a.z, p.b.dx, p.b.dy, p.b.dz,
                                p.a.E, p.d.kind, p.d.axial, p.d.mat, bp, L, G, S, lg, sb, bins, ctl, cnt, M, A)) {
            A.maxdraws = (unsigned long long)draws;
            A.maxhist = (unsigned long long)hist;
        }
    }
    flush_hist_acc(A, 0, cnt);
}

// Warp-cooperative finish for staged libraries: one WARP per queued particle
// carries it to death (k_finish's policy; a lone 272-nuclide fold runs 32
// nuclides per gather round instead of one).
__global__ void __launch_bounds__(128) k_finish_warp(const int32_t* __restrict__ q, int64_t n, BatchP bp, DLib L,
                                                     DGeom G, DSlots S, DLog lg, DSites sb, double* bins, Ctl* ctl,
                                                     unsigned long long* cnt, DMesh M)
{
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool lead = (threadIdx.x & 31u) == 0;
    HistAcc A;
    for (int64_t i = w0; i < n; i += nw) {
        const int32_t s = q[i];
        const PState p = S.ps[s];
        if (*(volatile int32_t*)&ctl->err) break;
        uint64_t rng = p.b.rng;
        int32_t draws = p.d.draws, ordc = p.d.ordctr, hist = p.d.histlog;
        if (transport_to_death<true>(s, p.d.gid, rng, draws, ordc, hist, p.a.x, p.a.y, p.a.z, p.b.dx, p.b.dy,
                                     p.b.dz, p.a.E, p.d.kind, p.d.axial, p.d.mat, bp, L, G, S, lg, sb, bins, ctl,
                                     cnt, M, A))
            break;
        A.maxdraws = max(A.maxdraws, (unsigned long long)draws);
        A.maxhist = max(A.maxhist, (unsigned long long)hist);
    }
    if (lead) flush_hist_acc(A, 0, cnt);
}

}  // namespace emc
