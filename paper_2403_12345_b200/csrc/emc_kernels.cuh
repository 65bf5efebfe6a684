// Event kernels of the transport loop (one launch per queue sweep).
// Reference: kernels.py (K:<line>), replication.py (R:).
//
// Queue structure per event iteration (host loop in emc_engine.cu):
//   q_look --sort(mat, E)--> k_lookup --> k_advance --+--> q_col  --> k_collision --+
//      ^                                              +--> q_cross --> k_crossing ---+
//      +------------------------- q_next (scatter / crossed / refilled) -----------+
// Every in-flight particle is in q_look at the start of an iteration; deaths
// refill their slot from the batch cursor inside k_collision (K:1191-1202).
// Particle state is one 128-byte PState line per slot; kernels move whole
// 32-byte sectors (P0..P3) with vector loads/stores.
#pragma once
#include "emc_device.cuh"

namespace emc {

// Minimum resident 256-thread blocks per SM for the event kernels: bounds
// their registers so enough warps are resident to hide the gather latency
// (measured: collision 80 -> 63 ms per C4 batch at 4 blocks/SM).
#ifndef EMC_ADV_MINB
#define EMC_ADV_MINB 2
#endif
#ifndef EMC_COL_MINB
#define EMC_COL_MINB 4
#endif

// Warp-uniform grid-stride loop: every lane of a warp runs the same number of
// iterations (warp-synchronous helpers need all 32 lanes); `valid` masks the
// tail.
#define EMC_WARP_LOOP(n)                                                                   \
    for (int64_t emc_base_ = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u),     \
                 emc_stride_ = (int64_t)gridDim.x * blockDim.x;                            \
         emc_base_ < (int64_t)(n); emc_base_ += emc_stride_)

// Prefetch the particle line this lane handles in the next grid-stride
// iteration into L2, so its load there waits on L2 rather than DRAM.
#ifndef EMC_PREFETCH
#define EMC_PREFETCH 1
#endif
__device__ __forceinline__ void prefetch_next_line(const int32_t* __restrict__ q, int64_t i, int64_t stride,
                                                   int64_t n, const PState* ps)
{
    if (EMC_PREFETCH && i + stride < n) {
        const PState* p = ps + __ldg(q + i + stride);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
    }
}

// queue_push that also stores the lookup sort key at the pushed position
__device__ __forceinline__ void queue_push_key(int32_t* q, unsigned int* count, int32_t slot, bool pred,
                                               uint32_t* keys, uint32_t key)
{
    unsigned int mask = __ballot_sync(kFull, pred);
    unsigned int rank = __popc(mask & ((1u << lane_id()) - 1u));
    unsigned int base = 0;
    if (lane_id() == 0 && mask) base = atomicAdd(count, (unsigned int)__popc(mask));
    base = __shfl_sync(kFull, base, 0);
    if (pred) {
        q[base + rank] = slot;
        if (keys) keys[base + rank] = key;
    }
}

// The advance's three queue pushes (collision, next lookup with its sort key,
// leakage) with their tail atomics issued by lanes 0, 1, 2 in ONE atomic
// instruction: the warp waits for one round trip instead of three.
#ifndef EMC_PUSH3
#define EMC_PUSH3 1
#endif
__device__ __forceinline__ void queue_push3(int32_t slot, int32_t* q0, unsigned int* c0, bool p0,
                                            int32_t* q1, unsigned int* c1, bool p1, uint32_t* keys, uint32_t key,
                                            int32_t* q2, unsigned int* c2, bool p2)
{
    const unsigned m0 = __ballot_sync(kFull, p0), m1 = __ballot_sync(kFull, p1), m2 = __ballot_sync(kFull, p2);
    const unsigned ln = lane_id(), below = (1u << ln) - 1u;
    const unsigned m = ln == 0 ? m0 : ln == 1 ? m1 : m2;
    unsigned int* cp = ln == 0 ? c0 : ln == 1 ? c1 : c2;
    unsigned base = 0;
    if (ln < 3 && m) base = atomicAdd(cp, (unsigned int)__popc(m));
    const unsigned b0 = __shfl_sync(kFull, base, 0), b1 = __shfl_sync(kFull, base, 1),
                   b2 = __shfl_sync(kFull, base, 2);
    if (p0) q0[b0 + __popc(m0 & below)] = slot;
    if (p1) {
        const unsigned at = b1 + __popc(m1 & below);
        q1[at] = slot;
        if (keys) keys[at] = key;
    }
    if (p2) q2[b2 + __popc(m2 & below)] = slot;
}

// Lookup-queue sort keys written at push time (energy-major key of
// k_sort_keys<true>): the kernels that put a particle on the next lookup
// queue know its energy and material, so the sort needs no separate gather
// pass over the particle lines.  keys == nullptr: not written.
struct QKeys {
    uint32_t* keys;
    int32_t ebin_bits, ebin_shift, mat_bits, fine_bits;
};

__device__ __forceinline__ uint32_t lookup_key(const DLib& L, const QKeys& K, double E, int32_t m)
{
    const uint32_t eb = (uint32_t)energy_bin(E, L);
    uint32_t k = (uint32_t)__ldg(L.mat_group + m);
    k = K.ebin_bits ? ((k << K.ebin_bits) | (eb >> K.ebin_shift)) : k;
    if (K.mat_bits) k = (k << K.mat_bits) | (uint32_t)m;
    if (K.fine_bits) {
        const uint64_t e64 = (uint64_t)__double_as_longlong(E);
        k = (k << K.fine_bits) | (uint32_t)((e64 >> (L.shift - K.fine_bits)) & ((1u << K.fine_bits) - 1u));
    }
    return k;
}

// ----------------------------------------------------------- sourcing ---

// systematic resampling index of particle g (transport.py:188-200)
__device__ __forceinline__ int64_t resample_index(int64_t g, int64_t n, int64_t ppb, double u)
{
    if (n >= ppb) {
        double v = floor(__ddiv_rn(__dmul_rn(__dadd_rn((double)g, u), (double)n), (double)ppb));
        int64_t i = (int64_t)v;
        return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
    }
    return g % n;
}

// K:926-996: initialise `slot` with particle g of this batch.  Returns false
// (and records the error) when the history cannot start.
__device__ __forceinline__ bool source_particle(int32_t slot, int64_t g, const BatchP& bp,
                                                const DLib& L, const DGeom& G, const DSrc& src,
                                                const DSlots& S, Ctl* ctl, int& clamps)
{
    uint64_t s;
    if (EMC_GSKIP) {
        s = lcg_gskip(bp.seed_b, (uint64_t)g);
    } else {
        uint64_t off = ((uint64_t)bp.batch * (uint64_t)bp.pmax + (uint64_t)g) * (uint64_t)kStride;
        s = lcg_skip(bp.seed, off);
    }
    if (g == bp.perturb_gid) s ^= 1ULL;
    int32_t draws = 0;
    P0 a; P1 b;
    if (bp.fixed_source) {
        // fixed surface source (extension): uniform on the
        // z = 0 face, inward direction with mu = u (uniform in [0,1)), energy
        // fixed or from the fission spectrum
        double u1 = draw(s, draws), u2 = draw(s, draws);
        a.x = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u1), 1.0), G.hp);
        a.y = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u2), 1.0), G.hp);
        a.z = 0.0;
        const double mu = draw(s, draws), phi = __dmul_rn(kTwoPi, draw(s, draws));
        const double sn = __dsqrt_rn(__dsub_rn(1.0, __dmul_rn(mu, mu)));
        b.dx = __dmul_rn(sn, emc_cos(phi));
        b.dy = __dmul_rn(sn, emc_sin(phi));
        b.dz = mu;
        if (bp.src_energy > 0.0) a.E = bp.src_energy;
        else {
            double ue = draw(s, draws);
            a.E = clamp_energy(__dmul_rn(-bp.fission_t, emc_log(__dsub_rn(1.0, ue))), L, clamps);
        }
    } else if (bp.batch0) {
        double x, y, cx = 0.0, cy = 0.0;
        if (G.lat_n > 1) {       // lattice extension: uniform over the fuel pins, then the pin's disk
            int64_t k = (int64_t)__dmul_rn(draw(s, draws), (double)G.n_pins);
            k = k > G.n_pins - 1 ? G.n_pins - 1 : k;
            cx = G.pin_xy[2 * k]; cy = G.pin_xy[2 * k + 1];
        }
        for (;;) {
            double u1 = draw(s, draws), u2 = draw(s, draws);
            x = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u1), 1.0), G.radius);
            y = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u2), 1.0), G.radius);
            if (__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)) < G.r2) break;
            if (draws >= kStride) { set_error(ctl, nullptr, ERR_STREAM_OVERLAP, g); return false; }
        }
        if (G.lat_n > 1) { x = __dadd_rn(cx, x); y = __dadd_rn(cy, y); }
        a.x = x; a.y = y;
        a.z = __dmul_rn(draw(s, draws), G.height);
        double ua = draw(s, draws), ub = draw(s, draws);
        isotropic(ua, ub, b.dx, b.dy, b.dz);
        double ue = draw(s, draws);
        a.E = clamp_energy(__dmul_rn(-bp.fission_t, emc_log(__dsub_rn(1.0, ue))), L, clamps);
    } else {
        int64_t i = resample_index(g, src.n, bp.pmax, src.u) - src.lo;
        if (i < 0) i += src.n;                       // wrapped window (distributed.exchange_bank)
        a.x = src.x[i]; a.y = src.y[i]; a.z = src.z[i]; a.E = src.E[i];
        b.dx = src.dx[i]; b.dy = src.dy[i]; b.dz = src.dz[i];
    }
    b.rng = s;
    P3 d;
    int32_t ax, mat;
    int kd = locate_point(a.x, a.y, a.z, G, ax, mat);
    d.gid = g; d.draws = draws; d.ordctr = 0; d.histlog = 0; d.axial = ax; d.mat = mat;
    d.surf = -1; d.kind = (int8_t)kd; d.pad = 0;
    PState& p = S.ps[slot];
    p.a = a; p.b = b; st_p3(&p.d, d);
    if (kd < 0) { set_error(ctl, nullptr, ERR_OUTSIDE_BOX, g); return false; }
    return true;
}

__global__ void k_source_init(BatchP bp, DLib L, DGeom G, DSrc src, DSlots S, int32_t n0,
                              int32_t* q, Ctl* ctl, unsigned long long* cnt, QKeys K)
{
    int clamps = 0; unsigned long long sourced = 0;
    EMC_WARP_LOOP(n0) {
        int64_t i = emc_base_ + lane_id();
        bool ok = false;
        uint32_t key = 0;
        if (i < n0) {
            ok = source_particle((int32_t)i, bp.g_lo + i, bp, L, G, src, S, ctl, clamps);
            sourced += 1;
            if (ok && K.keys) key = lookup_key(L, K, S.ps[i].a.E, S.ps[i].d.mat);
        }
        queue_push_key(q, &ctl->nL2, (int32_t)i, ok, K.keys, key);
    }
    warp_add_u64(cnt + CNT_SOURCED, sourced);
    warp_add_u64(cnt + CNT_CLAMPS, (unsigned long long)clamps);
}

// ----------------------------------------------------------------- sort ---

// Lookup-queue key: (composition group, energy band, material, energy bin).
// The sort only buys memory coherence for the lookup (physics is
// sort-invariant, acceptance criterion 1).  Material-uniform warps keep the
// density gathers uniform; bands (a coarse log-energy partition of the
// library range) make the whole GPU sweep one band of the grid at a time for
// all materials of a group, so the record working set stays cache-resident.
// The fine key is the log-hash bin (~half a grid spacing).
//
// ENERGY_MAJOR (used with the staged lookup): (group, energy bin, material).
// A chunk of ~1000 consecutive particles then spans a few grid records per
// nuclide (the staged windows), and the material key inside a bin makes the
// shared-memory density reads of a warp mostly broadcasts.
template <bool ENERGY_MAJOR>
__global__ void k_sort_keys(const int32_t* __restrict__ q, int32_t n, const PState* __restrict__ ps,
                            DLib L, uint32_t* __restrict__ keys, int ebin_bits, int ebin_shift, int mat_bits,
                            int band_bits, int n_bands)
{
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t s = q[i];
    const int32_t m = ps[s].d.mat;
    const uint32_t eb = (uint32_t)energy_bin(ps[s].a.E, L);
    uint32_t k = (uint32_t)__ldg(L.mat_group + m);
    if (ENERGY_MAJOR) {
        // band_bits = extra energy bits below the hash bin (warps of one
        // material then span a fraction of the bin: more broadcast reads)
        k = ebin_bits ? ((k << ebin_bits) | (eb >> ebin_shift)) : k;
        k = (k << mat_bits) | (uint32_t)m;
        if (band_bits) {
            const uint64_t eb64 = (uint64_t)__double_as_longlong(ps[s].a.E);
            k = (k << band_bits) | (uint32_t)((eb64 >> (L.shift - band_bits)) & ((1u << band_bits) - 1u));
        }
    } else {
        const uint32_t band = (uint32_t)(((uint64_t)eb * (uint64_t)n_bands) / (uint64_t)L.nbins);
        k = (k << band_bits) | band;
        k = (k << mat_bits) | (uint32_t)m;
        k = ebin_bits ? ((k << ebin_bits) | (eb >> ebin_shift)) : k;
    }
    keys[i] = k;
}

// Permute particle lines into sorted queue order (dst[i] = src[perm[i]]):
// one random 128-byte line read + one streamed write per particle, after
// which lookup/advance address slot i directly and crossing/collision walk
// near-monotone subsequences.  Physics is slot-invariant.
__global__ void __launch_bounds__(256) k_reorder(const int32_t* __restrict__ perm, int32_t n,
                                                 const PState* __restrict__ src, PState* __restrict__ dst)
{
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    dst[i] = src[perm[i]];
}

// --------------------------------------------------------------- lookup ---

// K:573-710: macroscopic sigma_t/c/f/nu-sigma_f at the particle's energy in
// its cell material, sequential fold in composition order.  One lane per
// particle (the fold order is part of the bit-exact contract); the queue is
// sorted so the 32 lanes of a warp share material and nearby grid brackets.
// One block of NT threads per residency slot: the grid-stride loop hands each
// block NT *consecutive* queue entries, so with NT = 1024 all 32 warps of an
// SM work on neighbouring particles (same material, adjacent energies) and
// share every grid record they gather through L1.
template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_lookup(const int32_t* __restrict__ q, int32_t n, DLib L,
                                                        DSlots S, int32_t fused, unsigned long long* cnt,
                                                        const unsigned int* nptr = nullptr)
{
    if (nptr) n = (int32_t)*nptr;        // tail mode: queue length lives on the device
    unsigned long long nl = 0;
    EMC_WARP_LOOP(n) {
        int64_t i = emc_base_ + lane_id();
        if (i < n) {
            int32_t s = q[i];
            double E = S.ps[s].a.E;
            int32_t m = S.ps[s].d.mat;
            P2 c;
            macro_tcf(L, m, E, c.t, c.c, c.f, c.nsf, fused ? ckpt_of(S, s) : nullptr, S.nck, S.ck_row);
            S.ps[s].c = c;
            nl += (unsigned long long)(__ldg(L.mat_off + m + 1) - __ldg(L.mat_off + m));
        }
    }
    warp_add_u64(cnt + CNT_INTERP_TRANSPORT, 4ull * nl);
    warp_add_u64(cnt + CNT_NUCLIDE_LOOKUPS, nl);
}

// Lookup through the union grid (accel = double_index / unionized): one
// thread per particle, like k_lookup.
template <bool MERGED>
__global__ void __launch_bounds__(256) k_lookup_union(const int32_t* __restrict__ q, int32_t n, DLib L, DUnion U,
                                                      DSlots S, int32_t fused, unsigned long long* cnt,
                                                      const unsigned int* nptr)
{
    if (nptr) n = (int32_t)*nptr;
    unsigned long long nl = 0;
    EMC_WARP_LOOP(n) {
        int64_t i = emc_base_ + lane_id();
        if (i < n) {
            int32_t s = q[i];
            double E = S.ps[s].a.E;
            int32_t m = S.ps[s].d.mat;
            P2 c;
            macro_tcf_union<MERGED>(L, U, m, E, c.t, c.c, c.f, c.nsf, fused ? ckpt_of(S, s) : nullptr, S.nck, S.ck_row);
            S.ps[s].c = c;
            nl += (unsigned long long)(__ldg(L.mat_off + m + 1) - __ldg(L.mat_off + m));
        }
    }
    warp_add_u64(cnt + CNT_INTERP_TRANSPORT, 4ull * nl);
    warp_add_u64(cnt + CNT_NUCLIDE_LOOKUPS, nl);
}

// Warp-per-particle lookup for the sparse tail of a batch: a lone fuel
// particle's 272-nuclide fold through the global path is ~272 dependent
// gathers long, which sets the duration of every small tail iteration.  Here
// the 32 lanes of a warp look up 32 nuclides of ONE particle at a time
// (independent gathers), then every lane replays the reference's sequential
// fold over those 32 values in composition order (shuffles; same operations,
// same order as macro_tcf, so bit-identical sums and checkpoints).
// LPP lanes per particle (32: one particle per warp; 8: four per warp for
// mid-size tails).  Trip counts are made warp-uniform (the warp's longest
// composition) so every shuffle is executed by all 32 lanes.
template <int LPP>
__global__ void __launch_bounds__(256) k_lookup_warp(const int32_t* __restrict__ q, int32_t n, DLib L, DSlots S,
                                                     int32_t fused, unsigned long long* cnt,
                                                     const unsigned int* nptr)
{
    constexpr int PPW = 32 / LPP;                 // particles per warp
    if (nptr) n = (int32_t)*nptr;
    const int lane = (int)(threadIdx.x & 31u), sub = lane % LPP, grpl = lane / LPP;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long nl = 0;
    for (int64_t ib = w0 * PPW; ib < n; ib += nw * PPW) {
        const int64_t i = ib + grpl;
        const bool have = i < n;
        int32_t s = 0, m = 0, e0 = 0, ncomp = 0, bin = 0;
        double E = 1.0;
        if (have) {
            s = q[i];
            E = S.ps[s].a.E;
            m = S.ps[s].d.mat;
            const int32_t grp = __ldg(L.mat_group + m);
            e0 = __ldg(L.grp_off + grp);
            ncomp = __ldg(L.grp_off + grp + 1) - e0;
            bin = energy_bin(E, L);
        }
        int32_t nmax = ncomp;
        for (int o = 16; o; o >>= 1) nmax = max(nmax, __shfl_xor_sync(kFull, nmax, o));
        double* const ck = (fused && have) ? ckpt_of(S, s) : nullptr;
        double st = 0.0, sc = 0.0, sf = 0.0, snf = 0.0;
        for (int32_t k0 = 0; k0 < nmax; k0 += LPP) {
            double t = 0.0, cc = 0.0, f = 0.0, den = 0.0, dn = 0.0;
            const int32_t k = k0 + sub;
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
            const int kn = min(LPP, nmax - k0);
            for (int j = 0; j < kn; ++j) {
                const double tj = __shfl_sync(kFull, t, j, LPP), cj = __shfl_sync(kFull, cc, j, LPP);
                const double fj = __shfl_sync(kFull, f, j, LPP), dj = __shfl_sync(kFull, den, j, LPP);
                const double dnj = __shfl_sync(kFull, dn, j, LPP);
                if (k0 + j < ncomp) {
                    st = __dadd_rn(st, __dmul_rn(dj, tj));
                    sc = __dadd_rn(sc, __dmul_rn(dj, cj));
                    sf = __dadd_rn(sf, __dmul_rn(dj, fj));
                    snf = __dadd_rn(snf, __dmul_rn(dnj, fj));
                    if (ck && sub == 0 && ((k0 + j + 1) & (kCkptStride - 1)) == 0) {
                        const int32_t row = (k0 + j + 1) / kCkptStride - 1;
                        if (row < S.nck) ck[(int64_t)row * S.ck_row] = st;
                    }
                }
            }
        }
        if (have && sub == 0) {
            P2 c; c.t = st; c.c = sc; c.f = sf; c.nsf = snf;
            S.ps[s].c = c;
            nl += (unsigned long long)(__ldg(L.mat_off + m + 1) - __ldg(L.mat_off + m));
        }
    }
    warp_add_u64(cnt + CNT_INTERP_TRANSPORT, 4ull * nl);
    warp_add_u64(cnt + CNT_NUCLIDE_LOOKUPS, nl);
}

// Lookup microbenchmark kernel (tools/lookup_micro.py via emc_bench_lookup,
// variant 4): the plain gather lookup (macro_tcf) over (mat, E) pairs; the
// staged production kernel is variant 8 (k_lookup_staged<1, ...>).
__global__ void __launch_bounds__(256, 4) k_lookup_bench(int32_t n, DLib L, const double* __restrict__ Es,
                                                         const int32_t* __restrict__ mats, double* __restrict__ out)
{
    EMC_WARP_LOOP(n) {
        int64_t i = emc_base_ + lane_id();
        if (i < n) {
            double st, sc, sf, snf;
            macro_tcf(L, mats[i], Es[i], st, sc, sf, snf, out + n + i, 16, n);
            out[i] = st + sc + sf + snf;
        }
    }
}

// -------------------------------------------------------------- advance ---

// tally scoring of one flight segment into the dense (region, score) bins
// (fast reduction): one warp reduction + atomic per distinct region in the
// warp for up to three regions (energy-major queues mix a few materials per
// warp), per-lane atomics for the rest.
//
// The five sums of a round are a reduce-scatter butterfly rather than five
// all-reduces: at xor 16 the lower half-warp keeps scores 0-2 and the upper
// 3-4, at xor 8 the 3-value quarters split {0,2}|{1} and the others {3}|{4},
// at xor 4 the one 2-value group splits; xor 2 and xor 1 finish.  8 f64
// shuffles instead of 25, and the five atomics are one instruction issued by
// lanes 0, 8, 4, 16, 24 (scores 0, 1, 2, 3, 4).
#ifndef EMC_SCORE_BFLY
#define EMC_SCORE_BFLY 1
#endif
#ifndef EMC_SCORE_ACC
#define EMC_SCORE_ACC 1
#endif
__device__ __forceinline__ void score_bins(double* bins, bool valid, int32_t base, const double v[5])
{
    unsigned todo = __ballot_sync(kFull, valid);
    const unsigned ln = lane_id();
    for (int round = 0; round < 3 && todo; ++round) {
        const int l = __ffs(todo) - 1;
        const int32_t b = __shfl_sync(kFull, base, l);
        const bool in = valid && base == b;
        todo &= ~__ballot_sync(kFull, in);
        if (EMC_SCORE_BFLY) {
            double x0 = in ? v[0] : 0.0, x1 = in ? v[1] : 0.0, x2 = in ? v[2] : 0.0;
            double x3 = in ? v[3] : 0.0, x4 = in ? v[4] : 0.0;
            const bool h16 = ln & 16, h8 = ln & 8, h4 = ln & 4;
            // xor 16: lower keeps (0,1,2), upper keeps (3,4,-)
            double a0 = (h16 ? x3 : x0) + __shfl_xor_sync(kFull, h16 ? x0 : x3, 16);
            double a1 = (h16 ? x4 : x1) + __shfl_xor_sync(kFull, h16 ? x1 : x4, 16);
            double a2 = (h16 ? 0.0 : x2) + __shfl_xor_sync(kFull, h16 ? x2 : 0.0, 16);
            // xor 8: keep (a0, a2) below, (a1, -) above
            double b0 = (h8 ? a1 : a0) + __shfl_xor_sync(kFull, h8 ? a0 : a1, 8);
            double b1 = (h8 ? 0.0 : a2) + __shfl_xor_sync(kFull, h8 ? a2 : 0.0, 8);
            // xor 4: keep b0 below, b1 above
            double c0 = (h4 ? b1 : b0) + __shfl_xor_sync(kFull, h4 ? b0 : b1, 4);
            c0 += __shfl_xor_sync(kFull, c0, 2);
            c0 += __shfl_xor_sync(kFull, c0, 1);
            // lane -> score: 0->0, 4->2, 8->1, 16->3, 24->4
            const int k = ln == 0 ? 0 : ln == 4 ? 2 : ln == 8 ? 1 : ln == 16 ? 3 : ln == 24 ? 4 : -1;
            if (k >= 0 && c0 != 0.0) atomicAdd(bins + b + k, c0);
        } else {
            #pragma unroll
            for (int k = 0; k < 5; ++k) {
                double s = warp_sum_f64(in ? v[k] : 0.0);
                if ((int)ln == l && s != 0.0) atomicAdd(bins + b + k, s);
            }
        }
        if (in) valid = false;
    }
    if (valid) {
        #pragma unroll
        for (int k = 0; k < 5; ++k) if (v[k] != 0.0) atomicAdd(bins + base + k, v[k]);
    }
}

// K:782-811: cross surface d.surf -- reflect on an outer box plane, nudge
// past the surface, update cell and material (in registers)
__device__ __forceinline__ void cross_surface(P0& a, P1& b, P3& d, const DGeom& G)
{
    const int32_t surf = d.surf;
    if (surf >= SURF_XMIN && surf <= SURF_ZMAX) {
        if (surf == SURF_XMIN || surf == SURF_XMAX) b.dx = -b.dx;
        else if (surf == SURF_YMIN || surf == SURF_YMAX) b.dy = -b.dy;
        else b.dz = -b.dz;
    }
    a.x = __dadd_rn(a.x, __dmul_rn(b.dx, kNudge));
    a.y = __dadd_rn(a.y, __dmul_rn(b.dy, kNudge));
    a.z = __dadd_rn(a.z, __dmul_rn(b.dz, kNudge));
    if (surf == SURF_CYL) {
        if (d.kind == KIND_FUEL) { d.kind = KIND_MOD; d.axial = -1; }
        else { d.kind = KIND_FUEL; d.axial = axial_index(a.z, G.n_axial, G.height); }
    } else if (surf >= SURF_AXIAL_BASE && surf < SURF_LATTICE) {
        int32_t jpl = surf - SURF_AXIAL_BASE;
        d.axial = b.dz > 0.0 ? jpl : jpl - 1;
    }
    d.mat = d.kind == KIND_FUEL ? G.fuel_mats[d.axial] : G.mod_mat;
}

// K:713-811: sample the flight distance, score the segment, move.
// Collisions go to q_col; surface crossings are completed here (the second
// half of the reference's advance) and go straight back to the lookup queue
// q_next -- except vacuum leakage, which k_crossing ends and refills.
//
// Same-material crossings (moderator -> moderator lattice planes, reflections
// on the outer box): the lookup the reference performs next would return the
// very same macroscopic cross sections (same material, same energy; the slot's
// sigma_t checkpoints were written by that same lookup and the slot does not
// move inside this kernel), so the particle takes its next flight here, up to
// kMaxChain segments per launch (3 since the chain's scores are reduced once
// per chain: C4 +1.6%, C3 +2.6%, C2 +6.6% over 2; 4 and 6 segments, or a
// minimum of 4 / 8 chaining lanes per warp, are not better; before the
// accumulation 2 was best: C4 +4.5% over no chains).  The skipped lookups are counted as the
// lookup events (and interpolations) they are in the reference; draws,
// scores, log ordinals and banked sites are exactly those of the unchained
// schedule (physics is schedule-invariant, acceptance criterion 1).
#ifndef EMC_ADV_CHAIN
#define EMC_ADV_CHAIN 3
#endif
constexpr int kMaxChain = EMC_ADV_CHAIN;
#ifndef EMC_ADV_CHAIN_MIN
#define EMC_ADV_CHAIN_MIN 1
#endif
constexpr int kChainMinLanes = EMC_ADV_CHAIN_MIN;   // a warp chains another round only if this many lanes want to

__global__ void __launch_bounds__(256, EMC_ADV_MINB) k_advance(const int32_t* __restrict__ q, int32_t n, BatchP bp,
                                                 DLib L, DGeom G, DSlots S, DLog lg, double* bins,
                                                 int32_t* q_col, int32_t* q_cross, Ctl* ctl,
                                                 unsigned long long* cnt, DMesh M, const unsigned int* nptr,
                                                 int32_t* q_next, QKeys K)
{
    if (nptr) n = (int32_t)*nptr;        // tail mode: queue length lives on the device
    unsigned long long interp_score = 0, chained = 0, chained_interp = 0;
    EMC_WARP_LOOP(n) {
        int64_t i = emc_base_ + lane_id();
        bool valid = i < n, to_col = false, to_cross = false, leak = false;
        int32_t s = valid ? q[i] : 0;
        prefetch_next_line(q, i, emc_stride_, n, S.ps);
        double kE = 1.0;                     // energy for the next lookup's sort key
        P0 a{}; P1 b{}; P2 c{}; P3 d{};
        if (valid) {
            const PState& p = S.ps[s];
            a = p.a; b = p.b; c = p.c; d = ld_p3(&p.d);
            if (!(c.t > 0.0)) {
                set_error(ctl, cnt, ERR_NONPOSITIVE_SIGMA, d.gid);
                valid = false;
            }
        }
        bool seg = valid;                    // this lane flies a segment this round
        bool moved = false;
        // fast-mode scores of a chain accumulate per lane while the region
        // stays and go out in one warp reduction after the chain (EMC_SCORE_ACC)
        double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        int32_t acc_base = -1;
        for (int rep = 0;; ++rep) {
            double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            int32_t base = 0;
            unsigned nlog = 0;
            bool again = false, scored = false;
            if (seg) {
                const double sig_t = c.t;
                const int32_t mat0 = d.mat;
                double u = draw(b.rng, d.draws);
                double d_coll = __ddiv_rn(-emc_log(__dsub_rn(1.0, u)), sig_t);
                int32_t surf;
                double dist = boundary_distance(a.x, a.y, a.z, b.dx, b.dy, b.dz, d.kind, d.axial, G, surf);
                if (surf < 0) {
                    set_error(ctl, cnt, ERR_NO_SURFACE, d.gid);
                    valid = false;
                    to_col = to_cross = false;
                } else {
                    bool crossing = !(d_coll < dist);
                    double ell = crossing ? dist : d_coll;
                    if (bp.score) {
                        int32_t region = d.kind == KIND_FUEL ? d.axial : G.n_axial;
                        base = region * 5;
                        double fl = __dmul_rn(1.0, ell);     // wt == 1 (analog, K:950)
                        if (bp.fused) {
                            v[1] = __dmul_rn(fl, sig_t);
                            v[2] = __dmul_rn(fl, __dadd_rn(c.c, c.f));
                            v[3] = __dmul_rn(fl, c.f);
                            v[4] = __dmul_rn(fl, c.nsf);
                        } else {   // K:757-765 naive re-assembly
                            double st2, sc2, sf2, snf2;
                            macro_tcf_simple(L, d.mat, a.E, st2, sc2, sf2, snf2, nullptr, 0);
                            interp_score += 3ull * (unsigned long long)(__ldg(L.mat_off + d.mat + 1) -
                                                                        __ldg(L.mat_off + d.mat));
                            v[1] = __dmul_rn(fl, st2);
                            v[2] = __dmul_rn(fl, __dadd_rn(sc2, sf2));
                            v[3] = __dmul_rn(fl, sf2);
                            v[4] = __dmul_rn(fl, snf2);
                        }
                        v[0] = fl;
                        #pragma unroll
                        for (int k = 0; k < 5; ++k) nlog += v[k] != 0.0;
                        if (M.on) score_mesh(M, a.x, a.y, a.z, b.dx, b.dy, b.dz, ell, sig_t);
                    }
                    a.x = __dadd_rn(a.x, __dmul_rn(b.dx, ell));
                    a.y = __dadd_rn(a.y, __dmul_rn(b.dy, ell));
                    a.z = __dadd_rn(a.z, __dmul_rn(b.dz, ell));
                    d.surf = (int16_t)surf;
                    moved = true;
                    if (d.draws >= kStride) {       // K:1159-1162
                        set_error(ctl, cnt, ERR_STREAM_OVERLAP, d.gid);
                        valid = false;
                        to_col = to_cross = false;
                    } else {
                        scored = true;
                        to_col = !crossing;
                        to_cross = crossing;
                        leak = crossing && G.vacuum && surf >= SURF_XMIN && surf <= SURF_ZMAX;
                        bool guarded = false;
                        if (crossing && !leak) cross_surface(a, b, d, G);
                        if (G.guard && !leak && box_guard(a.x, a.y, a.z, b.dx, b.dy, b.dz, G)) {
                            atomicAdd(cnt + CNT_BOX_GUARD, 1ull);      // rare: ~1e-9 per history
                            guarded = true;
                            to_col = false; to_cross = true;           // no collision here: re-look-up
                            if (G.vacuum) { leak = true; d.surf = SURF_XMIN; }
                            else {
                                int32_t ax, mt;
                                d.kind = (int8_t)locate_point(a.x, a.y, a.z, G, ax, mt);
                                d.axial = ax; d.mat = mt;
                            }
                        }
                        kE = a.E;
                        again = crossing && !leak && !guarded && d.mat == mat0 && rep + 1 < kMaxChain;
                    }
                }
            }
            if (bp.score && bp.use_logs) {
                unsigned want = scored ? nlog : 0u;
                unsigned long long at = warp_claim(&ctl->log_n, want);
                if (want) {
                    if (at + want > (unsigned long long)lg.cap) {
                        atomicExch(&ctl->ovf, 1);
                    } else {
                        unsigned j = 0;
                        #pragma unroll
                        for (int k = 0; k < 5; ++k) {
                            if (v[k] != 0.0) {
                                lg.gid[at + j] = d.gid; lg.ord[at + j] = d.ordctr + (int32_t)j;
                                lg.bin[at + j] = base + k; lg.val[at + j] = v[k];
                                ++j;
                            }
                        }
                    }
                    d.ordctr += (int32_t)want;
                    d.histlog += (int32_t)want;
                    if (d.histlog > kMaxHistLog) {
                        set_error(ctl, cnt, ERR_RUNAWAY_HISTORY, d.gid);
                        to_col = to_cross = false;
                        again = false;
                    }
                }
            } else if (bp.score) {
                if (EMC_SCORE_ACC) {
                    const bool flush = scored && acc_base >= 0 && base != acc_base;   // region changed
                    if (__any_sync(kFull, flush)) {
                        score_bins(bins, flush, acc_base, acc);
                        if (flush) {
                            #pragma unroll
                            for (int k = 0; k < 5; ++k) acc[k] = 0.0;
                            acc_base = -1;
                        }
                    }
                    if (scored) {
                        #pragma unroll
                        for (int k = 0; k < 5; ++k) acc[k] = __dadd_rn(acc[k], v[k]);
                        acc_base = base;
                    }
                } else {
                    score_bins(bins, scored, base, v);
                }
            }
            if (__popc(__ballot_sync(kFull, again)) < kChainMinLanes) {
                if (again) { to_col = false; to_cross = true; }   // back to the lookup queue instead
                break;
            }
            if (again) {       // the reference's next lookup, skipped: same material, same energy
                const unsigned long long nc = (unsigned long long)(__ldg(L.mat_off + d.mat + 1) -
                                                                   __ldg(L.mat_off + d.mat));
                chained += 1;
                chained_interp += 4ull * nc;
            }
            seg = again;
        }
        if (EMC_SCORE_ACC && bp.score && !bp.use_logs) score_bins(bins, acc_base >= 0, acc_base, acc);
        if (moved) { PState& p = S.ps[s]; p.a = a; p.b = b; }
        if (to_col || to_cross) st_p3(&S.ps[s].d, d);
        const bool to_next = to_cross && !leak;
        if (EMC_PUSH3) {
            queue_push3(s, q_col, &ctl->nC, to_col, q_next, &ctl->nL2, to_next, K.keys,
                        (to_next && K.keys) ? lookup_key(L, K, kE, d.mat) : 0u,
                        q_cross, &ctl->nX, G.vacuum && to_cross && leak);
        } else {
            queue_push(q_col, &ctl->nC, s, to_col);
            queue_push_key(q_next, &ctl->nL2, s, to_next, K.keys,
                           (to_next && K.keys) ? lookup_key(L, K, kE, d.mat) : 0u);
            if (G.vacuum) queue_push(q_cross, &ctl->nX, s, to_cross && leak);
        }
    }
    warp_add_u64(cnt + CNT_INTERP_SCORE, interp_score);
    warp_add_u64(cnt + CNT_EV_LOOKUP, chained);
    warp_add_u64(cnt + CNT_EV_ADVANCE, chained);
    warp_add_u64(cnt + CNT_INTERP_TRANSPORT, chained_interp);
}

// ---------------------------------------------------- surface crossing ---

// K:782-811 (second half of the reference advance): reflect on the outer
// box planes, nudge past the surface, update cell and material.  With vacuum
// boundaries (extension) an outer-plane crossing ends the history (leakage)
// and the slot is refilled from the batch cursor like a collision death.
__global__ void __launch_bounds__(256, EMC_COL_MINB) k_crossing(const int32_t* __restrict__ q, const unsigned int* nq,
                                                  BatchP bp, DLib L, DGeom G, DSrc src, DSlots S, int32_t* q_next,
                                                  Ctl* ctl, unsigned long long* cnt, QKeys K)
{
    const int32_t n = (int32_t)*nq;
    unsigned long long leaks = 0, sourced = 0, maxdraws = 0, maxhist = 0;
    int clamps = 0;
    EMC_WARP_LOOP(n) {
        int64_t i = emc_base_ + lane_id();
        bool valid = i < n, died = false;
        int32_t s = valid ? q[i] : 0;
        if (valid) {
            PState& p = S.ps[s];
            P0 a = p.a; P1 b = p.b; P3 d = ld_p3(&p.d);
            const int32_t surf = d.surf;
            if (surf >= SURF_XMIN && surf <= SURF_ZMAX && G.vacuum) {
                died = true;
                leaks += 1;
                maxdraws = max(maxdraws, (unsigned long long)d.draws);
                maxhist = max(maxhist, (unsigned long long)d.histlog);
            } else {                     // (k_advance completes non-leaking crossings itself)
                cross_surface(a, b, d, G);
                p.a = a; p.b = b; st_p3(&p.d, d);
            }
        }
        bool refill = false;
        if (G.vacuum) {          // warp-uniform: the claim below needs all lanes
            unsigned long long idx = warp_claim(&ctl->cursor, died ? 1u : 0u);
            if (died && idx < (unsigned long long)bp.n_assigned) {
                refill = source_particle(s, bp.g_lo + (int64_t)idx, bp, L, G, src, S, ctl, clamps);
                sourced += 1;
            }
        }
        const bool nxt = (valid && !died) || refill;
        queue_push_key(q_next, &ctl->nL2, s, nxt, K.keys,
                       (nxt && K.keys) ? lookup_key(L, K, S.ps[s].a.E, S.ps[s].d.mat) : 0u);
    }
    if (G.vacuum) {
        warp_add_u64(cnt + CNT_LEAKS, leaks);
        warp_add_u64(cnt + CNT_SOURCED, sourced);
        warp_add_u64(cnt + CNT_CLAMPS, (unsigned long long)clamps);
        warp_max_u64(cnt + CNT_MAX_DRAWS, maxdraws);
        warp_max_u64(cnt + CNT_MAX_HIST_LOG, maxhist);
    }
}

// ------------------------------------------------------------ collision ---

// Nuclide selection (K:841-884).  Fused: restart the cumulative walk from the
// last sigma_t prefix checkpoint <= target written by the lookup, so at most
// kCkptStride partials are re-interpolated (bit-identical to the stored
// part_t walk).  Naive: re-interpolate from the first nuclide (K:853-883).
// Optional first probe round of the checkpoint search: EMC_CK_WIN independent
// probes around the row the draw points at, g = floor(u * cmax) (tgt = u *
// sigma_t and the prefix grows about linearly in the checkpoint index for
// the benchmark libraries: the answer is in [g-1, g+3] for ~99% of
// collisions, measured offline on the C4 library), then the binary search on
// what is left.  The result is the same row whatever the probes (the
// predicate is monotone).  Measured SLOWER (C4 collision +10% at 6 probes,
// +9% at 4, +14% at 8): the queue is in slot order and every lane of a warp
// with the same material starts the binary search on the same row, so its
// first levels are coalesced loads (2 lines per warp) -- only its last ~3
// levels scatter, while every window probe is per-lane (a sector per lane).
// An evenly spaced K-ary round (same rows for the whole warp) then leaves K
// scattered probes instead of ~3: also slower.  Default 0: binary search.
#ifndef EMC_CK_WIN
#define EMC_CK_WIN 0
#endif
constexpr int kCkWin = EMC_CK_WIN;
__device__ __forceinline__ int32_t select_nuclide(const DLib& L, const double* ck, int32_t nck, int64_t cks,
                                                  int32_t e0,
                                                  int32_t e1, int32_t bin, double E, double u, double tgt,
                                                  bool fused, double& pt_sel, unsigned long long& interp)
{
    int32_t ncomp = e1 - e0;
    int32_t c = 0;
    double cum = 0.0;
    if (fused && ncomp > kCkptStride) {
        int32_t cmax = (ncomp - 1) / kCkptStride;
        if (cmax > nck) cmax = nck;
        int32_t lo = 0, hi = cmax;      // largest c with P_c <= tgt (P_0 = 0)
        if (kCkWin > 0 && cmax > 0) {
            const int32_t g = (int32_t)__dmul_rn(u, (double)cmax);
            const int32_t r0 = max(1, min(g - 1, cmax - kCkWin + 1));
            double pv[kCkWin > 0 ? kCkWin : 1];
            #pragma unroll
            for (int j = 0; j < kCkWin; ++j) pv[j] = ck[(int64_t)(min(r0 + j, cmax) - 1) * cks];
            #pragma unroll
            for (int j = 0; j < kCkWin; ++j) {
                const int32_t r = min(r0 + j, cmax);
                if (pv[j] <= tgt) lo = max(lo, r);
                else hi = min(hi, r - 1);
            }
        }
        while (lo < hi) {
            int32_t mid = (lo + hi + 1) >> 1;
            if (ck[(int64_t)(mid - 1) * cks] <= tgt) lo = mid; else hi = mid - 1;
        }
        c = lo;
        if (c > 0) cum = ck[(int64_t)(c - 1) * cks];
    }
    int32_t ksel = e1 - 1;
    pt_sel = 0.0;
    // walk in groups of SN nuclides, software-pipelined one group ahead: the
    // composition entries and hash bounds of group g+1 are loaded while the
    // records of group g are in flight, so each group costs one dependent
    // gather instead of three; the comparison walk stays sequential (same cum
    // and pt values as K:846-852)
#ifndef EMC_WALK_SN
#define EMC_WALK_SN 1
#endif
    constexpr int SN = EMC_WALK_SN;
    const int32_t kstart = e0 + c * kCkptStride;
    double nden[SN];
    int32_t ng0[SN], nlast[SN], nh[SN];
    #pragma unroll
    for (int u = 0; u < SN; ++u) {
        const Comp cc = load_comp(L.comp + min(kstart + u, e1 - 1));
        nden[u] = cc.den; ng0[u] = cc.g0; nlast[u] = cc.glen - 1;
        nh[u] = nlast[u] > 0 ? __ldg(L.hash + (int64_t)cc.nid * L.nbins + bin) : 0;
    }
    for (int32_t k0 = kstart; k0 < e1; k0 += SN) {
        double den[SN], e0v[SN], t0[SN], e1v[SN], t1[SN];
        int32_t st[SN], g0[SN], lastv[SN], hv[SN];
        #pragma unroll
        for (int u = 0; u < SN; ++u) { den[u] = nden[u]; g0[u] = ng0[u]; lastv[u] = nlast[u]; hv[u] = nh[u]; }
        #pragma unroll
        for (int u = 0; u < SN; ++u) {            // records of this group
            const Rec* __restrict__ R = L.rec + g0[u];
            const double2 p0 = *reinterpret_cast<const double2*>(&R[hv[u]].E);        // (E, t) of point i
            const double2 p1 = *reinterpret_cast<const double2*>(&R[min(hv[u] + 1, lastv[u])].E);
            e0v[u] = p0.x; t0[u] = p0.y; e1v[u] = p1.x; t1[u] = p1.y;
        }
        if (k0 + SN < e1) {                       // next group's entries and hash bounds
            #pragma unroll
            for (int u = 0; u < SN; ++u) {
                const Comp cc = load_comp(L.comp + min(k0 + SN + u, e1 - 1));
                nden[u] = cc.den; ng0[u] = cc.g0; nlast[u] = cc.glen - 1;
                nh[u] = nlast[u] > 0 ? __ldg(L.hash + (int64_t)cc.nid * L.nbins + bin) : 0;
            }
        }
        #pragma unroll
        for (int u = 0; u < SN; ++u) {
            const int32_t last = lastv[u];
            if (last == 0) { st[u] = 1; continue; }
            int32_t i = hv[u];
            if (e1v[u] <= E && i + 1 < last) {     // rare: bracket beyond the hashed lower bound
                const Rec* __restrict__ R = L.rec + g0[u];
                do {
                    ++i; e0v[u] = e1v[u]; t0[u] = t1[u];
                    const double2 q = *reinterpret_cast<const double2*>(&R[i + 1].E);
                    e1v[u] = q.x; t1[u] = q.y;
                } while (e1v[u] <= E && i + 1 < last);
            }
            st[u] = (i == 0 && E <= e0v[u]) ? 1 : (E >= e1v[u] ? 2 : 0);
        }
        #pragma unroll
        for (int u = 0; u < SN; ++u) {
            const int32_t k = k0 + u;
            if (k >= e1) break;
            const double mt = st[u] == 1 ? t0[u] : st[u] == 2 ? t1[u] : lerp(t0[u], t1[u], frac(E, e0v[u], e1v[u]));
            double pt = __dmul_rn(den[u], mt);
            if (!fused) interp += 1;
            pt_sel = pt;
            if (__dadd_rn(cum, pt) > tgt) { return k; }
            cum = __dadd_rn(cum, pt);
        }
    }
    return ksel;
}

// two warp claims in one atomic round trip: n0 entries per lane from cur0
// (lane 31 issues), one entry per lane with p1 from cur1 (lane 30 issues)
#ifndef EMC_COL_PREFETCH
#define EMC_COL_PREFETCH 0   // measured: collision +2% slower with it
#endif
#ifndef EMC_CLAIM2
#define EMC_CLAIM2 1
#endif
__device__ __forceinline__ void warp_claim2(unsigned long long* cur0, unsigned int n0, unsigned long long& at0,
                                            unsigned long long* cur1, bool p1, unsigned long long& at1)
{
    unsigned int incl = n0;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned int y = __shfl_up_sync(kFull, incl, o);
        if ((int)lane_id() >= o) incl += y;
    }
    const unsigned int total = __shfl_sync(kFull, incl, 31);
    const unsigned m1 = __ballot_sync(kFull, p1);
    const unsigned ln = lane_id();
    const unsigned int add = ln == 31 ? total : __popc(m1);
    unsigned long long base = 0;
    if (ln >= 30 && add) base = atomicAdd(ln == 31 ? cur0 : cur1, (unsigned long long)add);
    at0 = __shfl_sync(kFull, base, 31) + (incl - n0);
    at1 = __shfl_sync(kFull, base, 30) + (unsigned long long)__popc(m1 & ((1u << ln) - 1u));
}

// K:814-923 + refill (K:1187-1202)
__global__ void __launch_bounds__(256, EMC_COL_MINB) k_collision(const int32_t* __restrict__ q, const unsigned int* nq,
                                                   BatchP bp, DLib L, DGeom G, DSrc src, DSlots S,
                                                   DLog lg, DSites sb, double* bins, int32_t* q_next,
                                                   Ctl* ctl, unsigned long long* cnt, QKeys K)
{
    const int32_t n = (int32_t)*nq;
    unsigned long long interp = 0, captures = 0, fissions = 0, sourced = 0;
    unsigned long long maxdraws = 0, maxhist = 0;
    int clamps = 0;
    EMC_WARP_LOOP(n) {
        int64_t i = emc_base_ + lane_id();
        bool valid = i < n;
        int32_t s = valid ? q[i] : 0;
        if (EMC_COL_PREFETCH) prefetch_next_line(q, i, emc_stride_, n, S.ps);
        bool alive = false, died = false;
        double kval = 0.0;
        unsigned nsites = 0;
        P0 a{}; P1 b{}; P3 d{};
        if (valid) {
            PState& p = S.ps[s];
            a = p.a; b = p.b; d = ld_p3(&p.d);
            const P2 c = p.c;
            const double st = c.t;
            kval = __dmul_rn(1.0, __ddiv_rn(c.nsf, st));            // wt * (nsf / st)
            const double E = a.E;
            const int32_t e0 = __ldg(L.mat_off + d.mat), e1 = __ldg(L.mat_off + d.mat + 1);
            const int32_t bin = energy_bin(E, L);
            double u1 = draw(b.rng, d.draws);
            double tgt = __dmul_rn(u1, st);
            double pt_sel;
            int32_t ksel = select_nuclide(L, ckpt_of(S, s), S.nck, S.ck_row, e0, e1, bin, E, u1, tgt,
                                          bp.fused != 0, pt_sel, interp);
            const Comp cs = load_comp(L.comp + ksel);
            double s_s, s_c, s_f;
            micro_scf(L, cs, bin, E, s_s, s_c, s_f);
            interp += 3;
            double ps_ = __dmul_rn(cs.den, s_s), pc = __dmul_rn(cs.den, s_c);
            double u2 = draw(b.rng, d.draws);
            double tgt2 = __dmul_rn(u2, pt_sel);
            if (tgt2 < ps_) {                                    // scatter
                double u3 = draw(b.rng, d.draws), u4 = draw(b.rng, d.draws);
                isotropic(u3, u4, b.dx, b.dy, b.dz);
                double u5 = draw(b.rng, d.draws);
                double ep = __dmul_rn(E, __dadd_rn(bp.alpha, __dmul_rn(__dsub_rn(1.0, bp.alpha), u5)));
                a.E = clamp_energy(ep, L, clamps);
                alive = true;
            } else if (tgt2 < __dadd_rn(ps_, pc)) {             // capture
                captures += 1;
                died = true;
            } else {                                             // fission
                fissions += 1;
                died = true;
                double u5 = draw(b.rng, d.draws);
                double nu_sel = __ldg(L.nu + cs.nid);
                int64_t ns = (int64_t)floor(__dadd_rn(__ddiv_rn(nu_sel, bp.k_run), u5));
                nsites = ns > 0 ? (unsigned)ns : 0u;
            }
        }
        // contribution to the k-effective bin (every batch), K:829-834
        if (bp.use_logs) {
            unsigned want = (valid && kval != 0.0) ? 1u : 0u;
            unsigned long long at = warp_claim(&ctl->log_n, want);
            if (want) {
                if (at + 1 > (unsigned long long)lg.cap) atomicExch(&ctl->ovf, 1);
                else { lg.gid[at] = d.gid; lg.ord[at] = d.ordctr; lg.bin[at] = bp.kbin; lg.val[at] = kval; }
                d.ordctr += 1;
                d.histlog += 1;
                if (d.histlog > kMaxHistLog) { set_error(ctl, cnt, ERR_RUNAWAY_HISTORY, d.gid); alive = died = false; }
            }
        } else {
            warp_add_f64(bins + bp.kbin, valid ? kval : 0.0);
        }
        // fission sites (K:913-922); the site draws continue the parent stream.
        // Each site takes 3 draws, so the stream-overlap check (K:1183-1186)
        // is known here, and the site claim and the batch-cursor claim for
        // the dead slots go out as one atomic instruction (EMC_CLAIM2).
        const bool overlap = valid && (alive || died) && d.draws + 3 * (int32_t)nsites >= kStride;
        unsigned long long at, idx = 0;
        if (EMC_CLAIM2) {
            warp_claim2(&ctl->site_n, nsites, at, &ctl->cursor, died && !overlap, idx);
        } else {
            at = warp_claim(&ctl->site_n, nsites);
        }
        for (unsigned ms = 0; ms < nsites; ++ms) {
            double ua = draw(b.rng, d.draws), ub = draw(b.rng, d.draws);
            double sx, sy, sz;
            isotropic(ua, ub, sx, sy, sz);
            double uc = draw(b.rng, d.draws);
            double es = clamp_energy(__dmul_rn(-bp.fission_t, emc_log(__dsub_rn(1.0, uc))), L, clamps);
            unsigned long long w = at + ms;
            if (w >= (unsigned long long)sb.cap) { atomicExch(&ctl->ovf, 2); continue; }
            sb.parent[w] = d.gid; sb.ord[w] = (int32_t)ms;
            sb.x[w] = a.x; sb.y[w] = a.y; sb.z[w] = a.z;
            sb.dx[w] = sx; sb.dy[w] = sy; sb.dz[w] = sz; sb.E[w] = es;
        }
        if (overlap) {                                           // K:1183-1186
            set_error(ctl, cnt, ERR_STREAM_OVERLAP, d.gid);
            alive = died = false;
        }
        if (alive) {
            PState& p = S.ps[s];
            p.a = a; p.b = b; st_p3(&p.d, d);
        }
        bool refill = false;
        if (died) {                                              // K:999-1006
            maxdraws = max(maxdraws, (unsigned long long)d.draws);
            maxhist = max(maxhist, (unsigned long long)d.histlog);
        }
        // claim the next source particle for dead slots
        if (!EMC_CLAIM2) idx = warp_claim(&ctl->cursor, died ? 1u : 0u);
        if (died && idx < (unsigned long long)bp.n_assigned) {
            refill = source_particle(s, bp.g_lo + (int64_t)idx, bp, L, G, src, S, ctl, clamps);
            sourced += 1;
        }
        const bool nxt = alive || refill;
        queue_push_key(q_next, &ctl->nL2, s, nxt, K.keys,
                       !(nxt && K.keys) ? 0u : alive ? lookup_key(L, K, a.E, d.mat)
                                                     : lookup_key(L, K, S.ps[s].a.E, S.ps[s].d.mat));
    }
    warp_add_u64(cnt + CNT_INTERP_TRANSPORT, interp);
    warp_add_u64(cnt + CNT_CAPTURES, captures);
    warp_add_u64(cnt + CNT_FISSIONS, fissions);
    warp_add_u64(cnt + CNT_SOURCED, sourced);
    warp_add_u64(cnt + CNT_CLAMPS, (unsigned long long)clamps);
    warp_max_u64(cnt + CNT_MAX_DRAWS, maxdraws);
    warp_max_u64(cnt + CNT_MAX_HIST_LOG, maxhist);
}

}  // namespace emc

namespace emc {

// Tail mode (small queues, source exhausted): iterations run back to back
// without a host round trip.  Between iterations this one-thread kernel makes
// the queue pushed by the last crossing/collision sweeps the current one and
// keeps the event counters the host loop would have kept (K:1132-1206 counts).
__global__ void k_tail_begin(Ctl* ctl, unsigned long long* cnt)
{
    const unsigned int n = ctl->nL2;
    ctl->nLcur = n;
    ctl->nL2 = 0; ctl->nC = 0; ctl->nX = 0;
    if (n) {
        cnt[CNT_EV_LOOKUP] += n; cnt[CNT_EV_ADVANCE] += n;
        cnt[CNT_INV_LOOKUP] += 1; cnt[CNT_INV_ADVANCE] += 1;
    }
}

__global__ void k_tail_end(Ctl* ctl, unsigned long long* cnt)
{
    const unsigned int c = ctl->nC;
    if (c) { cnt[CNT_EV_COLLISION] += c; cnt[CNT_INV_COLLISION] += 1; }
}

}  // namespace emc
