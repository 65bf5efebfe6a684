// Batch-end kernels (canonical bank, deterministic log reduction) and the
// single-operation kernels behind the public API wrappers (macro_lookup,
// locate, distance_to_boundary, sample_isotropic, ...).
#pragma once
#include "emc_device.cuh"

namespace emc {

// ------------------------------------------------------ canonical bank ---

// key = (parent - g_lo) << 20 | ordinal: sorting by it reproduces the
// reference's lexsort((ordinal, parent)) (R:227) on this rank's gid block.
__global__ void k_bank_keys(const int64_t* __restrict__ parent, const int32_t* __restrict__ ord,
                            int64_t n, int64_t g_lo, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ idx)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = ((uint64_t)(parent[i] - g_lo) << 20) | (uint64_t)(uint32_t)ord[i];
    idx[i] = (int32_t)i;
}

// 32-bit (parent - g_lo, ordinal) keys when they fit (see emc_engine.cu)
__global__ void k_bank_keys32(const int64_t* __restrict__ parent, const int32_t* __restrict__ ord,
                              int64_t n, int64_t g_lo, int ord_bits, uint32_t* __restrict__ keys,
                              int32_t* __restrict__ idx)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = ((uint32_t)(parent[i] - g_lo) << ord_bits) | (uint32_t)ord[i];
    idx[i] = (int32_t)i;
}

__global__ void k_bank_gather(const int32_t* __restrict__ idx, int64_t n, DSites in, DSites out)
{
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int32_t i = idx[j];
    out.parent[j] = in.parent[i]; out.ord[j] = in.ord[i];
    out.x[j] = in.x[i]; out.y[j] = in.y[i]; out.z[j] = in.z[i];
    out.dx[j] = in.dx[i]; out.dy[j] = in.dy[i]; out.dz[j] = in.dz[i]; out.E[j] = in.E[i];
}

// ------------------------------------------- deterministic log reduction ---

// key = bin | (gid - g_lo) | ord.  Sorted by it, each bin's entries appear in
// the canonical (gid, emission) order of tally.py:79-89, so folding each bin
// segment left to right reproduces replay_into_bins (K:1219-1223) exactly.
__global__ void k_log_keys(const int64_t* __restrict__ gid, const int32_t* __restrict__ ord,
                           const int32_t* __restrict__ bin, int64_t n, int64_t g_lo, int gid_bits,
                           uint64_t* __restrict__ keys)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = ((uint64_t)bin[i] << (gid_bits + 17)) | ((uint64_t)(gid[i] - g_lo) << 17) |
              (uint64_t)(uint32_t)ord[i];
}

// one thread per bin: sequential left fold of its segment, starting from init
// One CTA per bin: the bin's value range (binary-searched in the sorted keys)
// is streamed through shared memory in tiles by the whole CTA (coalesced,
// double-buffered) while thread 0 runs the left fold -- the order-defining,
// inherently serial add chain -- out of shared memory.
constexpr int LF_THREADS = 256, LF_TILE = 2048;

__global__ void __launch_bounds__(LF_THREADS) k_log_fold(const uint64_t* __restrict__ keys,
                                                         const double* __restrict__ vals, int64_t n, int shift,
                                                         int32_t n_bins, const double* __restrict__ init,
                                                         double* __restrict__ out)
{
    __shared__ double tile[2][LF_TILE];
    __shared__ int64_t rng[2];
    const int32_t b = blockIdx.x;
    if (b >= n_bins) return;
    if (threadIdx.x < 2) {                     // [first key with bin >= b, first key with bin >= b + 1)
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if ((int64_t)(keys[mid] >> shift) < b + (int32_t)threadIdx.x) lo = mid + 1; else hi = mid;
        }
        rng[threadIdx.x] = lo;
    }
    __syncthreads();
    const int64_t r0 = rng[0], r1 = rng[1];
    double s = init[b];
    int buf = 0;
    for (int64_t j = r0 + threadIdx.x; j < min(r1, r0 + LF_TILE); j += LF_THREADS) tile[0][j - r0] = vals[j];
    __syncthreads();
    for (int64_t t0 = r0; t0 < r1; t0 += LF_TILE) {
        const int64_t t1 = min(r1, t0 + LF_TILE), n0 = t1 + LF_TILE;
        // the other threads fetch the next tile while thread 0 folds this one
        for (int64_t j = t1 + threadIdx.x; j < min(r1, n0); j += LF_THREADS) tile[buf ^ 1][j - t1] = vals[j];
        if (threadIdx.x == 0) {
            const double* v = tile[buf];
            const int m = (int)(t1 - t0);
            int k = 0;
            for (; k + 8 <= m; k += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[k + u]);
            }
            for (; k < m; ++k) s = __dadd_rn(s, v[k]);
        }
        __syncthreads();
        buf ^= 1;
    }
    if (threadIdx.x == 0) out[b] = s;
}

// stable replay key for reduce_batch(order="fast"): (bin, position)
__global__ void k_replay_keys(const int32_t* __restrict__ bin, int64_t n, int pos_bits,
                              uint64_t* __restrict__ keys)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = ((uint64_t)bin[i] << pos_bits) | (uint64_t)i;
}

// ----------------------------------------------------------- API kernels ---

// emc_grid_index: (clamp state, local bracket index) of composition entry k at E
__global__ void k_api_bracket(DLib L, int64_t n, const int32_t* __restrict__ entry,
                              const double* __restrict__ E, int32_t* __restrict__ out)
{
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const Comp c = L.comp[entry[q]];
    Rec r0, r1; int32_t gi;
    const int st = bracket(L, c, energy_bin(E[q], L), E[q], gi, r0, r1);
    out[2 * q] = st;
    out[2 * q + 1] = gi - c.g0;
}

// K:287-331 macro_lookup_full: five sums + per-entry (t, s, c, f) partials
template <int ACCEL>   // 0 log-hash (binary-search equivalent), 1 double_index, 2 unionized (X:292-318)
__global__ void k_api_macro(DLib L, DUnion U, int64_t n, const int32_t* __restrict__ mats,
                            const double* __restrict__ E, int32_t max_comp, double* __restrict__ sums,
                            double* __restrict__ parts)
{
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    int32_t m = mats[q];
    double e = E[q];
    int32_t e0 = L.mat_off[m], e1 = L.mat_off[m + 1];
    int32_t bin = energy_bin(e, L);
    const int64_t uj = ACCEL ? union_interval(U, L, e) : 0;
    double st = 0.0, ss = 0.0, sc = 0.0, sf = 0.0, snf = 0.0;
    for (int32_t k = e0; k < e1; ++k) {
        const Comp c = L.comp[k];
        double t, s, cc, f;
        if (ACCEL == 0) {
            Rec r0, r1; int32_t gi;
            int cl = bracket(L, c, bin, e, gi, r0, r1);
            if (cl) { t = r0.t; s = L.ch_s[gi]; cc = r0.c; f = r0.f; }
            else {
                double fr = frac(e, r0.E, r1.E);
                t = lerp(r0.t, r1.t, fr); s = lerp(L.ch_s[gi], L.ch_s[gi + 1], fr);
                cc = lerp(r0.c, r1.c, fr); f = lerp(r0.f, r1.f, fr);
            }
        } else {        // K:216-254: end clamps on the nuclide grid, then the mapped bracket
            const Rec* R = L.rec + c.g0;
            const int32_t last = c.glen - 1;
            if (e <= R[0].E) { t = R[0].t; s = L.ch_s[c.g0]; cc = R[0].c; f = R[0].f; }
            else if (e >= R[last].E) { t = R[last].t; s = L.ch_s[c.g0 + last]; cc = R[last].c; f = R[last].f; }
            else {
                const int32_t i = U.map[uj * U.n_nuc + c.nid];
                const Rec r0 = R[i], r1 = R[i + 1];
                const double fr = frac(e, r0.E, r1.E);
                if (ACCEL == 2) {
                    const double* mg = U.merged + (uj * U.n_nuc + c.nid) * 8;
                    t = lerp(mg[0], mg[1], fr); s = lerp(mg[2], mg[3], fr);
                    cc = lerp(mg[4], mg[5], fr); f = lerp(mg[6], mg[7], fr);
                } else {
                    t = lerp(r0.t, r1.t, fr); s = lerp(L.ch_s[c.g0 + i], L.ch_s[c.g0 + i + 1], fr);
                    cc = lerp(r0.c, r1.c, fr); f = lerp(r0.f, r1.f, fr);
                }
            }
        }
        double pt = __dmul_rn(c.den, t);
        st = __dadd_rn(st, pt);
        ss = __dadd_rn(ss, __dmul_rn(c.den, s));
        sc = __dadd_rn(sc, __dmul_rn(c.den, cc));
        sf = __dadd_rn(sf, __dmul_rn(c.den, f));
        snf = __dadd_rn(snf, __dmul_rn(c.dn, f));
        if (parts) {
            double* p = parts + (q * max_comp + (k - e0)) * 4;
            p[0] = pt; p[1] = __dmul_rn(c.den, s); p[2] = __dmul_rn(c.den, cc); p[3] = __dmul_rn(c.den, f);
        }
    }
    double* o = sums + q * 5;
    o[0] = st; o[1] = ss; o[2] = sc; o[3] = sf; o[4] = snf;
}

__global__ void k_api_locate(DGeom G, int64_t n, const double* __restrict__ pos, int32_t* __restrict__ out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t ax, mat;
    int kd = locate_point(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], G, ax, mat);
    out[3 * i] = kd; out[3 * i + 1] = ax; out[3 * i + 2] = mat;
}

__global__ void k_api_distance(DGeom G, int64_t n, const double* __restrict__ pos,
                               const double* __restrict__ dir, const int32_t* __restrict__ cell,
                               double* __restrict__ dist, int32_t* __restrict__ surf)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t sf;
    dist[i] = boundary_distance(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], dir[3 * i], dir[3 * i + 1],
                                dir[3 * i + 2], cell[2 * i], cell[2 * i + 1], G, sf);
    surf[i] = sf;
}

// transport.py:161-174: isotropic direction / collision distance from a state
__global__ void k_api_particle_ops(int64_t n, const uint64_t* __restrict__ states,
                                   const double* __restrict__ sigma_t, double* __restrict__ iso,
                                   double* __restrict__ dcol, uint64_t* __restrict__ st_iso,
                                   uint64_t* __restrict__ st_dcol)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t s = states[i];
    int32_t d = 0;
    double u1 = draw(s, d), u2 = draw(s, d);
    isotropic(u1, u2, iso[3 * i], iso[3 * i + 1], iso[3 * i + 2]);
    st_iso[i] = s;
    s = states[i];
    double u = draw(s, d);
    dcol[i] = __ddiv_rn(-emc_log(__dsub_rn(1.0, u)), sigma_t[i]);
    st_dcol[i] = s;
}

// raw transcendental replicas (parity harness for emc_libm.h on the device)
__global__ void k_api_libm(int64_t n, const double* __restrict__ x, double* __restrict__ out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = x[i];
    out[3 * i] = emc_log(v);
    out[3 * i + 1] = emc_sin(v);
    out[3 * i + 2] = emc_cos(v);
}

// division check: out[2i] = n/d through the precomputed reciprocal (staged
// lookup path), out[2i+1] = the IEEE division
__global__ void k_api_div(int64_t n, const double* __restrict__ num, const double* __restrict__ den,
                          double* __restrict__ out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a = num[i], b = den[i];
    out[2 * i] = div_by_rcp(a, b, div_rcp(b));
    out[2 * i + 1] = __ddiv_rn(a, b);
}

__global__ void k_api_lcg_skip(int64_t n, const uint64_t* __restrict__ s, const uint64_t* __restrict__ k,
                               uint64_t* __restrict__ out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = lcg_skip(s[i], k[i]);
}

}  // namespace emc
