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

// One particle from "awaiting its cross-section lookup" to death, event after
// event (the loop body of run_history_batch, K:1055-1086, with the event
// kernels' arithmetic).  Returns true when the history failed (error set).
__device__ __forceinline__ bool transport_to_death(int32_t s, int64_t g, uint64_t& rng, int32_t& draws,
                                                   int32_t& ordc, int32_t& hist, double x, double y, double z,
                                                   double dx, double dy, double dz, double E, int kd, int32_t ax,
                                                   int32_t m, const BatchP& bp, const DLib& L, const DGeom& G,
                                                   const DSlots& S, const DLog& lg, const DSites& sb, double* bins,
                                                   Ctl* ctl, unsigned long long* cnt, const DMesh& M, HistAcc& A)
{
    double* ck = S.ckpt + s;
    for (;;) {
        // --- lookup (K:573-710)
        double st, sc, sf, snf;
        macro_tcf(L, m, E, st, sc, sf, snf, bp.fused ? ck : nullptr, S.nck, S.nslots);
        A.interp += 4ull * (unsigned long long)(L.mat_off[m + 1] - L.mat_off[m]);
        A.nuc_lookups += (unsigned long long)(L.mat_off[m + 1] - L.mat_off[m]);
        A.ev_l += 1;
        // --- advance (K:713-811)
        A.ev_a += 1;
        if (!(st > 0.0)) { set_error(ctl, cnt, ERR_NONPOSITIVE_SIGMA, g); return true; }
        double u = draw(rng, draws);
        double d_coll = __ddiv_rn(-emc_log(__dsub_rn(1.0, u)), st);
        int32_t surf;
        double dist = boundary_distance(x, y, z, dx, dy, dz, kd, ax, G, surf);
        if (surf < 0) { set_error(ctl, cnt, ERR_NO_SURFACE, g); return true; }
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
                    unsigned long long at = atomicAdd(&ctl->log_n, 1ULL);
                    if (at >= (unsigned long long)lg.cap) atomicExch(&ctl->ovf, 1);
                    else { lg.gid[at] = g; lg.ord[at] = ordc; lg.bin[at] = base + k; lg.val[at] = v[k]; }
                    ordc += 1; hist += 1;
                } else {
                    atomicAdd(bins + base + k, v[k]);
                }
            }
            if (hist > kMaxHistLog) { set_error(ctl, cnt, ERR_RUNAWAY_HISTORY, g); return true; }
            if (M.on) score_mesh(M, x, y, z, dx, dy, dz, ell, st);
        }
        x = __dadd_rn(x, __dmul_rn(dx, ell));
        y = __dadd_rn(y, __dmul_rn(dy, ell));
        z = __dadd_rn(z, __dmul_rn(dz, ell));
        bool died = false, guarded = false;
        if (!crossing && G.guard && box_guard(x, y, z, dx, dy, dz, G)) {   // box guard (extension)
            atomicAdd(cnt + CNT_BOX_GUARD, 1ull);
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
                atomicAdd(cnt + CNT_BOX_GUARD, 1ull);
                if (G.vacuum) { A.leaks += 1; died = true; }
                else kd = locate_point(x, y, z, G, ax, m);
            }
        } else {
            // --- collision (K:814-923)
            A.ev_c += 1;
            double kval = __dmul_rn(1.0, __ddiv_rn(snf, st));
            if (bp.use_logs) {
                if (kval != 0.0) {
                    unsigned long long at = atomicAdd(&ctl->log_n, 1ULL);
                    if (at >= (unsigned long long)lg.cap) atomicExch(&ctl->ovf, 1);
                    else { lg.gid[at] = g; lg.ord[at] = ordc; lg.bin[at] = bp.kbin; lg.val[at] = kval; }
                    ordc += 1; hist += 1;
                    if (hist > kMaxHistLog) { set_error(ctl, cnt, ERR_RUNAWAY_HISTORY, g); return true; }
                }
            } else {
                atomicAdd(bins + bp.kbin, kval);
            }
            int32_t e0 = L.mat_off[m], e1 = L.mat_off[m + 1];
            int32_t bin = energy_bin(E, L);
            double u1 = draw(rng, draws);
            double tgt = __dmul_rn(u1, st);
            double pt_sel;
            int32_t ksel = select_nuclide(L, ck, S.nck, S.nslots, e0, e1, bin, E, tgt, bp.fused != 0, pt_sel, A.interp);
            const Comp cs = L.comp[ksel];
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
                    unsigned long long at = atomicAdd(&ctl->site_n, (unsigned long long)ns);
                    for (int64_t ms = 0; ms < ns; ++ms) {
                        double ua = draw(rng, draws), ub = draw(rng, draws), sx, sy, sz;
                        isotropic(ua, ub, sx, sy, sz);
                        double uc = draw(rng, draws);
                        double es = clamp_energy(__dmul_rn(-bp.fission_t, emc_log(__dsub_rn(1.0, uc))), L, A.clamps);
                        unsigned long long w = at + ms;
                        if (w >= (unsigned long long)sb.cap) { atomicExch(&ctl->ovf, 2); continue; }
                        sb.parent[w] = g; sb.ord[w] = (int32_t)ms;
                        sb.x[w] = x; sb.y[w] = y; sb.z[w] = z;
                        sb.dx[w] = sx; sb.dy[w] = sy; sb.dz[w] = sz; sb.E[w] = es;
                    }
                }
            }
        }
        if (draws >= kStride) { set_error(ctl, cnt, ERR_STREAM_OVERLAP, g); return true; }
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

}  // namespace emc
