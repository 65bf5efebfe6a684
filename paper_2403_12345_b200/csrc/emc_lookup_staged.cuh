// Shared-memory-staged macroscopic cross-section lookup (K:573-710), sm_100a.
//
// The lookup queue is sorted by (composition group, log-hash energy bin,
// material), so the ~1000 particles one CTA takes (a "chunk") share a
// composition group and span a narrow energy range: for every nuclide of the
// group, all their brackets lie in a window of a few grid records (2-3 at the
// C4 population).  One producer warp streams, nuclide by nuclide and LK_D
// stages ahead, each window plus the row of material densities for that
// composition position into shared memory with bulk async copies
// (cp.async.bulk, completion on an mbarrier); 31 consumer warps, one lane per
// particle, run the reference's sequential fold over the group's nuclides out
// of shared memory.  The dependent global gathers (hash -> record) of the
// plain kernel disappear from the per-lane critical path; what is left per
// (particle, nuclide) is two shared-memory reads and the FP64 arithmetic.
//
// Arithmetic, fold order and bracket semantics are exactly macro_tcf's (and
// thus the reference's): windows only change where a record is read from.
// Windows wider than LK_R records (sparse populations at the tail of a batch)
// fall back to the global hash + scan path for that (chunk, nuclide), which is
// warp-uniform.
#pragma once
#include <algorithm>
#include "emc_device.cuh"

namespace emc {

// CTA = NW warps: NW-1 consumer warps (one particle per lane; a chunk is
// (NW-1)*32 consecutive queue entries) + 1 producer warp; MINB CTAs per SM.
constexpr int LK_G = 8;                    // nuclides per pipeline stage
#ifndef EMC_LK_FAST_UNROLL
#define EMC_LK_FAST_UNROLL 8
#endif
constexpr int kLkFastUnroll = EMC_LK_FAST_UNROLL;   // unroll of the stage fast path's nuclide loop
#ifndef EMC_LK_D
#define EMC_LK_D 3
#endif
constexpr int LK_D = EMC_LK_D;             // stages in flight (3: two CTAs fit per SM; 6 for one)
constexpr int LK_R = 16;                   // staged interval records per nuclide window
constexpr int LK_SCAN = 4;                 // wider windows start the scan at the hash bound
#ifndef EMC_LK_MIN_NUC
#define EMC_LK_MIN_NUC 16
#endif
constexpr int LK_MIN_NUC = EMC_LK_MIN_NUC;  // smaller groups use the direct path
constexpr int LK_DS = 2 * LK_G + 2;        // doubles per material in a density block: 8 (den, den*nu)
                                           // pairs; the 144-byte stride spreads materials over banks
constexpr int LK_DEN_BYTES_MAX = 150 * 1024;

enum : int32_t { LK_STAGED = 0, LK_GLOBAL = 1, LK_POINT = 2 };

struct __align__(16) LkMeta {
    int32_t lo, cnt, last, mode;   // window = interval records [lo, lo+cnt) of the nuclide; last = glen-1
    double nu;                     // nu of the nuclide (den*nu is formed per lane, K:632 order)
    int32_t g0, hrow;              // global fallback
};

// Per-(chunk, nuclide) meta word: window size (bits 0-4), mode (5-6),
// "edge" (7) = the window touches the nuclide's first or last grid point, the
// only case in which the reference's end clamps (K:600-612) can apply.  The
// consumers' fast path is exactly `word <= 4`: a staged window of <= 3
// intervals away from both grid ends -- no clamp tests, no scan.
__host__ __device__ constexpr uint32_t lk_word(int32_t cnt, int32_t mode, int32_t lo, int32_t last)
{
    return (uint32_t)(cnt & 31) | ((uint32_t)mode << 5) | ((uint32_t)(lo == 0 || lo + cnt - 1 >= last) << 7);
}

struct __align__(128) LkShared {
    unsigned long long full[LK_D], empty[LK_D];
    int32_t grp, bmin, bmax, pad;
    uint32_t word[LK_D][LK_G];
    uint32_t sfast[LK_D];          // pipelined kernel: every nuclide of the stage takes the fast path
    uint32_t pad2[(4 - LK_D % 4) % 4];
    longlong2 hdr[LK_D][LK_G];     // pipelined kernel, fast nuclides: bit patterns of E0[lo+1], E0[lo+2]
    LkMeta meta[LK_D][LK_G];
    IvRec iv[LK_D][LK_G][LK_R];
};

// A nuclide whose chunk window is staged, at most 3 intervals wide and at
// least one record away from both grid ends takes the pipelined kernel's fast
// path: the producer then copies exactly 4 records (lo..lo+3, all inside the
// grid) and publishes E0[lo+1], E0[lo+2] in the stage header.  Every chunk
// energy E has its bracket i in [lo, lo+cnt-2] and E < E0[i+1]; records past
// the window are real grid records with larger energies, so
//   li = [E0[lo+1] <= E] + [E0[lo+2] <= E]
// is exactly i - lo with no clamp, and neither end clamp (K:600-612) can apply.
__host__ __device__ constexpr bool lk_fast(int32_t mode, int32_t cnt, int32_t lo, int32_t last)
{
    return mode == LK_STAGED && cnt <= 4 && lo >= 1 && lo + 3 < last;
}

// density block of one stage: [n_mat][LK_DS] doubles
__host__ __device__ constexpr size_t lk_den_block(int n_mat) { return (size_t)n_mat * LK_DS * sizeof(double); }

__host__ __device__ constexpr size_t lk_smem_bytes(int n_mat, int den_staged)
{
    return sizeof(LkShared) + (den_staged ? (size_t)LK_D * lk_den_block(n_mat) : 0);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* b)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(b))
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, uint32_t bytes)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_addr(b)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(unsigned long long* b, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

// a wait that cannot complete is a bug: report it and trap instead of hanging
// the device (try_wait suspends for a while per call, so ~2^26 calls is far
// beyond any legitimate wait)
__device__ __noinline__ void mbar_stuck(const unsigned long long* b, uint32_t parity, uint32_t tag)
{
    printf("emc: mbarrier wait stuck: block %d thread %d smem 0x%x parity %u tag 0x%x\n", (int)blockIdx.x,
           (int)threadIdx.x, smem_addr(b), parity, tag);
    __trap();
}

__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity, uint32_t tag = 0)
{
    uint32_t spins = 0;
    while (!mbar_try_wait(b, parity)) {
        if (++spins == (1u << 26)) mbar_stuck(b, parity, tag);
    }
}

// global -> shared bulk copy (16-byte aligned, size a multiple of 16),
// completing `bytes` of transaction count on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ int warp_min_i32(int v)
{
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ int warp_max_i32(int v)
{
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Interval records: built once per library upload from the point records.
__global__ void k_build_intervals(const Rec* __restrict__ rec, const int64_t* __restrict__ grid_off, int32_t n_nuc,
                                  IvRec* __restrict__ iv)
{
    const int32_t nid = blockIdx.y;
    if (nid >= n_nuc) return;
    const int64_t a = grid_off[nid], b = grid_off[nid + 1];
    for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
        const Rec p = rec[i];
        IvRec v;
        v.E0 = p.E; v.t0 = p.t; v.c0 = p.c; v.f0 = p.f;
        if (i + 1 < b) {
            const Rec q = rec[i + 1];
            v.r = div_rcp(__dsub_rn(q.E, p.E));
            v.dt = __dsub_rn(q.t, p.t);
            v.dc = __dsub_rn(q.c, p.c);
            v.df = __dsub_rn(q.f, p.f);
        } else {
            v.r = 0.0; v.dt = 0.0; v.dc = 0.0; v.df = 0.0;
        }
        iv[i] = v;
    }
}

// (t, c, f) of one nuclide from global point records (hash + scan): the
// fallback for windows that did not fit a stage (same values as macro_tcf).
__device__ __forceinline__ void lk_micro_global(const DLib& L, int32_t g0, int32_t last, int32_t hrow, int32_t bin,
                                                double E, double& t, double& cc, double& f)
{
    const Rec* __restrict__ R = L.rec + g0;
    int32_t i = __ldg(L.hash + hrow + bin);
    Rec r0 = R[i], r1 = R[i + 1];
    while (r1.E <= E && i + 1 < last) { ++i; r0 = r1; r1 = R[i + 1]; }
    if (i == 0 && E <= r0.E) { t = r0.t; cc = r0.c; f = r0.f; }
    else if (E >= r1.E) { t = r1.t; cc = r1.c; f = r1.f; }
    else {
        const double fr = frac(E, r0.E, r1.E);
        t = lerp(r0.t, r1.t, fr);
        cc = lerp(r0.c, r1.c, fr);
        f = lerp(r0.f, r1.f, fr);
    }
}

// a <= b for positive doubles (energies): integer compare of the bit patterns
// keeps the bracket tests off the FP64 pipe
__device__ __forceinline__ bool pos_le(double a, double b)
{
    return __double_as_longlong(a) <= __double_as_longlong(b);
}

// Every case the fast path does not take: a staged window near a grid end
// (clamps, K:600-612) or wider than 3 intervals (scan from the hash bound),
// a 1-point nuclide, or a (chunk, nuclide) served from global memory.
__device__ __forceinline__ void lk_micro_slow(const DLib& L, const LkMeta& mt, uint32_t wd, const IvRec* W, double a1,
                                           double a2, int32_t bin, double E, double& tt, double& cc, double& ff)
{
    const int32_t cnt_ = (int32_t)(wd & 31u), mode = (int32_t)((wd >> 5) & 3u);
    if (mode == LK_POINT) {
        tt = W[0].t0; cc = W[0].c0; ff = W[0].f0;
        return;
    }
    if (mode == LK_GLOBAL) {
        lk_micro_global(L, mt.g0, mt.last, mt.hrow, bin, E, tt, cc, ff);
        return;
    }
    int32_t li;
    if (cnt_ <= 4) {
        li = min((int32_t)(a1 <= E) + (int32_t)(a2 <= E), cnt_ - 2);
    } else {
        // the reference's scan (hash bound, then forward while grid[i+1] <= E)
        // ends at the last record <= E of the ascending grid: count them in the
        // staged window (warp-uniform trip count, broadcast shared loads)
        li = 0;
        for (int32_t j = 1; j <= cnt_ - 2; ++j) li += (int32_t)pos_le(W[j].E0, E);
    }
    const double e0v = W[li].E0, e1 = W[li + 1].E0;
    const bool lo_clamp = mt.lo + li == 0 && E <= e0v, hi_clamp = e1 <= E;
    if (lo_clamp || hi_clamp) {
        const IvRec& b = hi_clamp && !lo_clamp ? W[li + 1] : W[li];
        tt = b.t0; cc = b.c0; ff = b.f0;
    } else {
        const IvRec& a = W[li];
        const double fr = div_by_rcp_safe(__dsub_rn(E, e0v), __dsub_rn(e1, e0v), a.r);
        tt = __dadd_rn(a.t0, __dmul_rn(fr, a.dt));
        cc = __dadd_rn(a.c0, __dmul_rn(fr, a.dc));
        ff = __dadd_rn(a.f0, __dmul_rn(fr, a.df));
    }
}

// One producer lane's view of nuclide k of the current pass.
struct LkNext {
    LkMeta mt;
    bool valid;
    bool fast;                     // lk_fast (pipelined kernel only)
    long long a1, a2;              // E0[lo+1], E0[lo+2] bit patterns when fast
};

template <bool HDR = false>
__device__ __forceinline__ void lk_prefetch(const DLib& L, int32_t e0, int32_t k, int32_t ncomp, int32_t bmin,
                                            int32_t bmax, LkNext& nx)
{
    nx.valid = k < ncomp;
    nx.fast = false;
    if (!nx.valid) return;
    const NucRef r = L.gnuc[e0 + k];
    LkMeta& mt = nx.mt;
    mt.last = r.glen - 1; mt.g0 = r.g0; mt.hrow = r.hrow; mt.nu = __ldg(L.nu + r.nid);
    if (mt.last == 0) {
        mt.mode = LK_POINT; mt.lo = 0; mt.cnt = 1;
    } else if (!__ldg(L.nsafe + r.nid)) {
        mt.mode = LK_GLOBAL; mt.lo = 0; mt.cnt = 0;
    } else {
        const int32_t lo = __ldg(L.hash + r.hrow + bmin);
        const int32_t hi = bmax + 1 < L.nbins ? __ldg(L.hash + r.hrow + bmax + 1) : mt.last - 1;
        mt.lo = lo;
        mt.cnt = hi - lo + 2;            // intervals lo..hi plus record hi+1 (<= last)
        mt.mode = mt.cnt <= LK_R ? LK_STAGED : LK_GLOBAL;
        if (HDR && lk_fast(mt.mode, mt.cnt, lo, mt.last)) {
            nx.fast = true;
            nx.a1 = __double_as_longlong(__ldg(&L.iv[r.g0 + lo + 1].E0));
            nx.a2 = __double_as_longlong(__ldg(&L.iv[r.g0 + lo + 2].E0));
        }
    }
}

// MODE 0: transport (queue q of slots, writes PState.c and the sigma_t
//         checkpoints); MODE 1: microbenchmark over (bE, bM), writes
//         bout[i] = st + sc + sf + snf and checkpoints at bout + n.
// PPL particles per consumer lane (adjacent queue entries): the stage's meta
// word, window energies and control flow are shared by the lane's particles,
// and their independent folds give the scheduler instruction-level
// parallelism to cover the shared-memory latency.
template <int MODE, bool DEN_ST, int NW, int MINB, int PPL>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_lookup_staged(const int32_t* __restrict__ q, int32_t n, DLib L, DSlots S, int32_t fused,
                    unsigned long long* cnt, const double* __restrict__ bE, const int32_t* __restrict__ bM,
                    double* __restrict__ bout, const unsigned int* nptr, PState* __restrict__ rdst)
{
    if (nptr) n = (int32_t)*nptr;        // tail mode: queue length lives on the device
    extern __shared__ __align__(128) unsigned char lk_raw[];
    LkShared& sh = *reinterpret_cast<LkShared*>(lk_raw);
    double* const sden = reinterpret_cast<double*>(lk_raw + sizeof(LkShared));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int LK_CONS = NW - 1, LK_CHUNK = LK_CONS * 32 * PPL;
    const bool producer = warp == LK_CONS;
    const int32_t nmat = L.n_mat;
    const int32_t nck = MODE == 0 ? S.nck : 16;

    if (threadIdx.x == 0) {
        for (int d = 0; d < LK_D; ++d) {
            mbar_init(&sh.full[d], 32);
            mbar_init(&sh.empty[d], LK_CONS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    uint32_t T = 0;                 // pipeline stage counter, identical in every thread
    unsigned long long nl = 0;
    for (int64_t base = (int64_t)blockIdx.x * LK_CHUNK; base < n; base += (int64_t)gridDim.x * LK_CHUNK) {
        int64_t i[PPL];
        bool pend[PPL];
        int32_t s[PPL], m[PPL], grp[PPL], bin[PPL];
        double E[PPL];
#pragma unroll
        for (int p = 0; p < PPL; ++p) {
            i[p] = base + (int64_t)threadIdx.x * PPL + p;
            pend[p] = !producer && i[p] < n;
            s[p] = 0; m[p] = 0; grp[p] = 0; bin[p] = 0; E[p] = 1.0;
            if (pend[p]) {
                if (MODE == 0 && rdst) {
                    // fused reorder (replaces k_reorder): move the particle's line to
                    // queue position i, which becomes its slot from here on
                    const PState line = S.ps[q[i[p]]];
                    rdst[i[p]] = line;
                    s[p] = (int32_t)i[p];
                    E[p] = line.a.E;
                    m[p] = line.d.mat;
                } else if (MODE == 0) {
                    s[p] = q[i[p]];
                    E[p] = S.ps[s[p]].a.E;
                    m[p] = S.ps[s[p]].d.mat;
                } else {
                    E[p] = bE[i[p]];
                    m[p] = bM[i[p]];
                }
                grp[p] = __ldg(L.mat_group + m[p]);
                bin[p] = energy_bin(E[p], L);
            }
        }
        // particles of small groups (< LK_MIN_NUC nuclides: the moderator) are
        // done right here, lane by lane, without the block-wide pass machinery
        {
            const bool ckon0 = MODE == 1 || fused;
            const int64_t cks0 = MODE == 0 ? S.ck_row : (int64_t)n;
#pragma unroll
            for (int p = 0; p < PPL; ++p) {
                if (pend[p] && __ldg(L.grp_off + grp[p] + 1) - __ldg(L.grp_off + grp[p]) < LK_MIN_NUC) {
                    double t0, c0, f0, n0;
                    macro_tcf(L, m[p], E[p], t0, c0, f0, n0,
                              ckon0 ? (MODE == 0 ? ckpt_of(S, s[p]) : bout + n + i[p]) : nullptr, nck, cks0);
                    if (MODE == 0) {
                        P2 c; c.t = t0; c.c = c0; c.f = f0; c.nsf = n0;
                        (rdst ? rdst : S.ps)[s[p]].c = c;
                    } else {
                        bout[i[p]] = t0 + c0 + f0 + n0;
                    }
                    nl += (unsigned long long)(__ldg(L.mat_off + m[p] + 1) - __ldg(L.mat_off + m[p]));
                    pend[p] = false;
                }
            }
        }
        // one pass per composition group present in the chunk (normally one)
        for (;;) {
            if (threadIdx.x == 0) { sh.grp = INT32_MAX; sh.bmin = INT32_MAX; sh.bmax = -1; }
            __syncthreads();
            {
                int g = INT32_MAX;
#pragma unroll
                for (int p = 0; p < PPL; ++p) g = min(g, pend[p] ? grp[p] : INT32_MAX);
                g = warp_min_i32(g);
                if (lane == 0 && g != INT32_MAX) atomicMin(&sh.grp, g);
            }
            __syncthreads();
            const int32_t G = sh.grp;
            if (G == INT32_MAX) break;
            bool mine[PPL], any = false;
            {
                int b0 = INT32_MAX, b1 = -1;
#pragma unroll
                for (int p = 0; p < PPL; ++p) {
                    mine[p] = pend[p] && grp[p] == G;
                    any |= mine[p];
                    if (mine[p]) { b0 = min(b0, bin[p]); b1 = max(b1, bin[p]); }
                }
                b0 = warp_min_i32(b0);
                b1 = warp_max_i32(b1);
                if (lane == 0 && b1 >= 0) { atomicMin(&sh.bmin, b0); atomicMax(&sh.bmax, b1); }
            }
            __syncthreads();
            const int32_t bmin = sh.bmin, bmax = sh.bmax;
            const int32_t e0 = __ldg(L.grp_off + G), ncomp = __ldg(L.grp_off + G + 1) - e0;
            double st[PPL], sc[PPL], sf[PPL], snf[PPL];
#pragma unroll
            for (int p = 0; p < PPL; ++p) { st[p] = 0.0; sc[p] = 0.0; sf[p] = 0.0; snf[p] = 0.0; }
            // sigma_t checkpoints: row r of particle p at ckb[r * cks] (formed at
            // the store, not kept live through the nuclide loop)
            const bool ckon = MODE == 1 || fused;
            const int64_t cks = MODE == 0 ? S.ck_row : (int64_t)n;
            const int nst = (ncomp + LK_G - 1) / LK_G;

            if (ncomp < LK_MIN_NUC) {
#pragma unroll
                for (int p = 0; p < PPL; ++p)
                    if (mine[p])
                        macro_tcf(L, m[p], E[p], st[p], sc[p], sf[p], snf[p],
                                  ckon ? (MODE == 0 ? ckpt_of(S, s[p]) : bout + n + i[p]) : nullptr, nck, cks);
            } else if (producer) {
                // lane j < LK_G owns nuclide 8t+j of every stage; its global
                // reads for stage t+1 are issued before it waits for slot t
                LkNext nx;
                nx.valid = false;
                if (lane < LK_G) lk_prefetch(L, e0, lane, ncomp, bmin, bmax, nx);
                for (int t = 0; t < nst; ++t, ++T) {
                    const int d = (int)(T % LK_D);
                    const LkNext cur = nx;
                    if (lane < LK_G && t + 1 < nst) lk_prefetch(L, e0, (t + 1) * LK_G + lane, ncomp, bmin, bmax, nx);
                    if (T >= (uint32_t)LK_D) mbar_wait(&sh.empty[d], ((T / LK_D) - 1) & 1);
                    uint32_t bytes = 0;
                    const bool copy_iv = lane < LK_G && cur.valid && cur.mt.mode != LK_GLOBAL;
                    if (lane < LK_G && cur.valid) {
                        sh.meta[d][lane] = cur.mt;
                        sh.word[d][lane] = lk_word(cur.mt.cnt, cur.mt.mode, cur.mt.lo, cur.mt.last);
                    }
                    if (copy_iv) bytes += (uint32_t)cur.mt.cnt * (uint32_t)sizeof(IvRec);
                    if (DEN_ST && lane == 0) bytes += (uint32_t)lk_den_block(nmat);
                    // expect before issuing so the phase cannot complete early
                    mbar_arrive_tx(&sh.full[d], bytes);
                    if (copy_iv)
                        bulk_g2s(&sh.iv[d][lane][0], L.iv + cur.mt.g0 + cur.mt.lo,
                                 (uint32_t)cur.mt.cnt * (uint32_t)sizeof(IvRec), &sh.full[d]);
                    if (DEN_ST && lane == 0)
                        bulk_g2s(sden + (size_t)d * nmat * LK_DS, L.denS + (size_t)t * nmat * LK_DS,
                                 (uint32_t)lk_den_block(nmat), &sh.full[d]);
                }
            } else {
                // a lane's particles outside this pass's group compute on a copy
                // of a member's (energy, bin, material) -- their windows would
                // not hold their brackets -- and their results are discarded
                double Eu[PPL];
                int32_t bu[PPL], mu[PPL];
                {
                    int32_t pm = 0;
#pragma unroll
                    for (int p = PPL - 1; p >= 0; --p) if (mine[p]) pm = p;
#pragma unroll
                    for (int p = 0; p < PPL; ++p) {
                        Eu[p] = mine[p] ? E[p] : E[pm];
                        bu[p] = mine[p] ? bin[p] : bin[pm];
                        mu[p] = mine[p] ? m[p] : m[pm];
                    }
                }
                for (int t = 0; t < nst; ++t, ++T) {
                    const int d = (int)(T % LK_D);
                    mbar_wait(&sh.full[d], (T / LK_D) & 1);
                    if (any) {
                        // staged group lists are whole stages (padded at upload)
#pragma unroll
                        for (int j = 0; j < LK_G; ++j) {
                            const int k = t * LK_G + j;
                            const uint32_t wd = sh.word[d][j];
                            const IvRec* W = sh.iv[d][j];
                            // issued with the meta word (always in-bounds shared memory)
                            const double a1 = W[1].E0, a2 = W[2].E0;
                            double tt[PPL], cc[PPL], ff[PPL];
                            if (__builtin_expect(wd <= 4u, 1)) {
                                // <= 3 interior intervals: li = #{j in 1..cnt-2 : E0_j <= E}
                                // (grids ascend; entries past the window are stale, hence
                                // the clamp to cnt-2).  Away from the grid ends E lies in
                                // [E0, E1) of interval li: no clamp can apply.
#pragma unroll
                                for (int p = 0; p < PPL; ++p) {
                                    const int32_t li =
                                        min((int32_t)(a1 <= Eu[p]) + (int32_t)(a2 <= Eu[p]), (int32_t)wd - 2);
                                    const double2 er = *reinterpret_cast<const double2*>(&W[li].E0);   // (E0, r)
                                    const double e1 = W[li + 1].E0;
                                    const IvRec& a = W[li];
                                    const double fr =
                                        div_by_rcp_safe(__dsub_rn(Eu[p], er.x), __dsub_rn(e1, er.x), er.y);
                                    tt[p] = __dadd_rn(a.t0, __dmul_rn(fr, a.dt));
                                    cc[p] = __dadd_rn(a.c0, __dmul_rn(fr, a.dc));
                                    ff[p] = __dadd_rn(a.f0, __dmul_rn(fr, a.df));
                                }
                            } else {
#pragma unroll
                                for (int p = 0; p < PPL; ++p)
                                    lk_micro_slow(L, sh.meta[d][j], wd, W, a1, a2, bu[p], Eu[p], tt[p], cc[p], ff[p]);
                            }
#pragma unroll
                            for (int p = 0; p < PPL; ++p) {
                                const double2 dd =
                                    DEN_ST ? *reinterpret_cast<const double2*>(sden + ((size_t)d * nmat + mu[p]) * LK_DS + 2 * j)
                                           : *reinterpret_cast<const double2*>(&L.ddT[(int64_t)k * nmat + mu[p]]);
                                st[p] = __dadd_rn(st[p], __dmul_rn(dd.x, tt[p]));
                                sc[p] = __dadd_rn(sc[p], __dmul_rn(dd.x, cc[p]));
                                sf[p] = __dadd_rn(sf[p], __dmul_rn(dd.x, ff[p]));
                                snf[p] = __dadd_rn(snf[p], __dmul_rn(dd.y, ff[p]));
                            }
                            if constexpr (kCkptStride < LK_G) {   // checkpoints inside the stage
                                if (ckon && (j + 1) % kCkptStride == 0 && k + 1 <= ncomp) {
                                    const int32_t row = (k + 1) / kCkptStride - 1;
#pragma unroll
                                    for (int p = 0; p < PPL; ++p) {
                                        double* ckb = MODE == 0 ? ckpt_of(S, s[p]) : bout + n + i[p];
                                        if (mine[p] && row < nck) ckb[(int64_t)row * cks] = st[p];
                                    }
                                }
                            }
                        }
                        // prefix checkpoint after every kCkptStride nuclides (whole stages)
                        static_assert(kCkptStride % LK_G == 0 || LK_G % kCkptStride == 0, "checkpoint stride");
                        constexpr int CKS = kCkptStride >= LK_G ? kCkptStride / LK_G : 1;
                        if (kCkptStride >= LK_G && ckon && (t + 1) % CKS == 0 && (t + 1) * LK_G <= ncomp) {
                            const int32_t row = (t + 1) / CKS - 1;
#pragma unroll
                            for (int p = 0; p < PPL; ++p) {
                                double* ckb = MODE == 0 ? ckpt_of(S, s[p]) : bout + n + i[p];
                                if (mine[p] && row < nck) ckb[(int64_t)row * cks] = st[p];
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sh.empty[d]);
                }
            }
#pragma unroll
            for (int p = 0; p < PPL; ++p) {
                if (mine[p]) {
                    if (MODE == 0) {
                        P2 c; c.t = st[p]; c.c = sc[p]; c.f = sf[p]; c.nsf = snf[p];
                        (rdst ? rdst : S.ps)[s[p]].c = c;
                    } else {
                        bout[i[p]] = st[p] + sc[p] + sf[p] + snf[p];
                    }
                    nl += (unsigned long long)(__ldg(L.mat_off + m[p] + 1) - __ldg(L.mat_off + m[p]));
                    pend[p] = false;
                }
            }
            __syncthreads();
        }
    }
    if (MODE == 0 && !producer) {
        warp_add_u64(cnt + CNT_INTERP_TRANSPORT, 4ull * nl);
        warp_add_u64(cnt + CNT_NUCLIDE_LOOKUPS, nl);
    }
}

// ---------------------------------------------------------------------------
// Chunk-pipelined variant (sorted queues).  The producer warp plans chunk c's
// passes (composition groups and energy-bin ranges) from the SORTED push-time
// keys instead of waiting for the consumers to load their particles and
// reduce over the block, publishes the plan in a two-slot descriptor ring
// (mbarriers, no __syncthreads in the chunk loop) and streams chunk c+1's
// first stages while the consumers are still folding chunk c.  Consumers check
// their own (group, bin) against the plan; a particle no pass covers (small
// groups, more than LK_MAXP groups in a chunk, or keys that do not match the
// particle) takes the per-lane global path, so correctness never depends on
// the keys -- only the speed does.
constexpr int LK_MAXP = 4;

struct LkKeys {
    const uint32_t* keys;          // sorted keys, aligned with the queue
    int32_t grp_shift;             // key >> grp_shift = composition group
    int32_t eb_shift;              // (key >> eb_shift) & eb_mask = energy bin >> ebin_shift
    uint32_t eb_mask;
    int32_t ebin_shift;
};

struct __align__(16) LkPipe {
    unsigned long long dfull[2], dempty[2];
    int32_t npass[2];
    int32_t G[2][LK_MAXP], bmin[2][LK_MAXP], bmax[2][LK_MAXP];
};

__host__ __device__ constexpr size_t lk_pipe_offset(int n_mat, int den_staged)
{
    return (lk_smem_bytes(n_mat, den_staged) + 15) & ~(size_t)15;
}

template <int MODE, bool DEN_ST, int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_lookup_piped(const int32_t* __restrict__ q, int32_t n, DLib L, DSlots S, int32_t fused,
                   unsigned long long* cnt, const double* __restrict__ bE, const int32_t* __restrict__ bM,
                   double* __restrict__ bout, PState* __restrict__ rdst, LkKeys K)
{
    constexpr int LK_CONS = NW - 1, LK_CHUNK = LK_CONS * 32;
    extern __shared__ __align__(128) unsigned char lk_raw[];
    LkShared& sh = *reinterpret_cast<LkShared*>(lk_raw);
    double* const sden = reinterpret_cast<double*>(lk_raw + sizeof(LkShared));
    const int32_t nmat = L.n_mat;
    LkPipe& P = *reinterpret_cast<LkPipe*>(lk_raw + lk_pipe_offset(nmat, DEN_ST));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = warp == LK_CONS;
    const int32_t nck = MODE == 0 ? S.nck : 16;
    const bool ckon = MODE == 1 || fused;
    const int64_t cks = MODE == 0 ? S.ck_row : (int64_t)n;

    if (threadIdx.x == 0) {
        for (int d = 0; d < LK_D; ++d) {
            mbar_init(&sh.full[d], 32);
            mbar_init(&sh.empty[d], LK_CONS);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&P.dfull[k], 1);
            mbar_init(&P.dempty[k], LK_CONS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    uint32_t T = 0;                 // pipeline stage counter (same sequence in every warp)
    uint32_t c = 0;                 // chunk counter of this CTA
    unsigned long long nl = 0;
    for (int64_t base = (int64_t)blockIdx.x * LK_CHUNK; base < n; base += (int64_t)gridDim.x * LK_CHUNK, ++c) {
        const int slot = (int)(c & 1u);
        const uint32_t use = c >> 1;
        if (producer) {
            // ---- plan: group runs of the sorted chunk -> passes
            if (c >= 2) mbar_wait(&P.dempty[slot], (use - 1) & 1, 0x40000u | c);
            const int64_t end = min(base + (int64_t)LK_CHUNK, (int64_t)n);
            int np = 0;
            int64_t s0 = base;
            while (s0 < end && np < LK_MAXP) {
                const uint32_t ka = __ldg(K.keys + s0);
                const uint32_t g = ka >> K.grp_shift;
                int64_t e = end;
                if ((__ldg(K.keys + end - 1) >> K.grp_shift) != g) {
                    for (int64_t j0 = s0 + 1; j0 < end; j0 += 32) {
                        const int64_t j = j0 + lane;
                        const bool brk = j < end && (__ldg(K.keys + j) >> K.grp_shift) != g;
                        const unsigned bal = __ballot_sync(0xffffffffu, brk);
                        if (bal) { e = j0 + __ffs(bal) - 1; break; }
                    }
                }
                const uint32_t kb = __ldg(K.keys + e - 1);
                const int32_t ncomp = __ldg(L.grp_off + g + 1) - __ldg(L.grp_off + g);
                if (ncomp >= LK_MIN_NUC) {
                    const int32_t lo = (int32_t)(((ka >> K.eb_shift) & K.eb_mask) << K.ebin_shift);
                    const int32_t hi = min((int32_t)(((((kb >> K.eb_shift) & K.eb_mask) + 1) << K.ebin_shift) - 1),
                                           L.nbins - 1);
                    if (lane == 0) { P.G[slot][np] = (int32_t)g; P.bmin[slot][np] = lo; P.bmax[slot][np] = hi; }
                    ++np;
                }
                s0 = e;
            }
            if (lane == 0) {
                P.npass[slot] = np;
                mbar_arrive(&P.dfull[slot]);     // release: the plan is visible to the waiting consumers
            }
            __syncwarp();
            // ---- stream the passes' stages (lane j < LK_G owns nuclide 8t+j)
            for (int p = 0; p < np; ++p) {
                const int32_t G = P.G[slot][p], bmin = P.bmin[slot][p], bmax = P.bmax[slot][p];
                const int32_t e0 = __ldg(L.grp_off + G), ncomp = __ldg(L.grp_off + G + 1) - e0;
                const int nst = (ncomp + LK_G - 1) / LK_G;
                LkNext nx;
                nx.valid = false;
                nx.fast = false;
                if (lane < LK_G) lk_prefetch<true>(L, e0, lane, ncomp, bmin, bmax, nx);
                for (int t = 0; t < nst; ++t, ++T) {
                    const int d = (int)(T % LK_D);
                    const LkNext cur = nx;
                    if (lane < LK_G && t + 1 < nst)
                        lk_prefetch<true>(L, e0, (t + 1) * LK_G + lane, ncomp, bmin, bmax, nx);
                    if (T >= (uint32_t)LK_D) mbar_wait(&sh.empty[d], ((T / LK_D) - 1) & 1, 0x10000u | T);
                    uint32_t bytes = 0;
                    const bool copy_iv = lane < LK_G && cur.valid && cur.mt.mode != LK_GLOBAL;
                    const bool fast = lane < LK_G && cur.valid && cur.fast;
                    const uint32_t ncopy = fast ? 4u : (uint32_t)cur.mt.cnt;
                    if (lane < LK_G && cur.valid) {
                        sh.meta[d][lane] = cur.mt;
                        sh.word[d][lane] = lk_word(cur.mt.cnt, cur.mt.mode, cur.mt.lo, cur.mt.last);
                        if (fast) sh.hdr[d][lane] = make_longlong2(cur.a1, cur.a2);
                    }
                    const unsigned fb = __ballot_sync(0xffffffffu, fast);
                    if (lane == 0) sh.sfast[d] = (fb & ((1u << LK_G) - 1u)) == ((1u << LK_G) - 1u);
                    if (copy_iv) bytes += ncopy * (uint32_t)sizeof(IvRec);
                    if (DEN_ST && lane == 0) bytes += (uint32_t)lk_den_block(nmat);
                    mbar_arrive_tx(&sh.full[d], bytes);
                    if (copy_iv)
                        bulk_g2s(&sh.iv[d][lane][0], L.iv + cur.mt.g0 + cur.mt.lo, ncopy * (uint32_t)sizeof(IvRec),
                                 &sh.full[d]);
                    if (DEN_ST && lane == 0)
                        bulk_g2s(sden + (size_t)d * nmat * LK_DS, L.denS + (size_t)t * nmat * LK_DS,
                                 (uint32_t)lk_den_block(nmat), &sh.full[d]);
                }
            }
            continue;
        }

        // ---- consumers: load the particle (fused reorder) while the plan is made
        const int64_t i = base + (int64_t)threadIdx.x;
        bool pend = i < n;
        int32_t s = 0, m = 0, grp = -1, bin = 0;
        double E = 1.0;
        if (pend) {
            if (MODE == 0 && rdst) {
                const PState line = S.ps[q[i]];
                rdst[i] = line;
                s = (int32_t)i;
                E = line.a.E;
                m = line.d.mat;
            } else if (MODE == 0) {
                s = q[i];
                E = S.ps[s].a.E;
                m = S.ps[s].d.mat;
            } else {
                E = bE[i];
                m = bM[i];
            }
            grp = __ldg(L.mat_group + m);
            bin = energy_bin(E, L);
        }
        mbar_wait(&P.dfull[slot], use & 1, 0x30000u | c);
        const int np = P.npass[slot];
        int pidx = -1;
        for (int p = 0; p < np; ++p)
            if (pidx < 0 && grp == P.G[slot][p] && bin >= P.bmin[slot][p] && bin <= P.bmax[slot][p]) pidx = p;
        if (pend && pidx < 0) {
            // not covered by a pass: small group (the moderator) or an odd chunk
            double t0, c0, f0, n0;
            macro_tcf(L, m, E, t0, c0, f0, n0, ckon ? (MODE == 0 ? ckpt_of(S, s) : bout + n + i) : nullptr, nck, cks);
            if (MODE == 0) {
                P2 cc; cc.t = t0; cc.c = c0; cc.f = f0; cc.nsf = n0;
                (rdst ? rdst : S.ps)[s].c = cc;
            } else {
                bout[i] = t0 + c0 + f0 + n0;
            }
            nl += (unsigned long long)(__ldg(L.mat_off + m + 1) - __ldg(L.mat_off + m));
            pend = false;
        }
        for (int p = 0; p < np; ++p) {
            const int32_t G = P.G[slot][p];
            const int32_t ncomp = __ldg(L.grp_off + G + 1) - __ldg(L.grp_off + G);
            const int nst = (ncomp + LK_G - 1) / LK_G;
            const bool mine = pend && pidx == p;
            const bool any = __any_sync(0xffffffffu, mine);
            // lanes outside the pass compute on a member's copy (results discarded)
            const int src_lane = any ? __ffs(__ballot_sync(0xffffffffu, mine)) - 1 : 0;
            // (the shuffles are executed by every lane: a full-mask shuffle under
            // a lane-dependent condition is undefined)
            const double Es = __shfl_sync(0xffffffffu, E, src_lane);
            const int32_t bs = __shfl_sync(0xffffffffu, bin, src_lane);
            const int32_t ms = __shfl_sync(0xffffffffu, m, src_lane);
            const double Eu = mine ? E : Es;
            const int32_t bu = mine ? bin : bs;
            const int32_t mu = mine ? m : ms;
            double st = 0.0, sc = 0.0, sf = 0.0, snf = 0.0;
// fast-path bracket compares: FP64 compares of the header energies (1) or
// integer compares of their bit patterns (0); identical for the positive
// finite grid energies here; measured lookup -0.7% with FP64 (fewer live
// registers around the header loads)
#ifndef EMC_LK_HDR_F64
#define EMC_LK_HDR_F64 1
#endif
            const long long Eb = __double_as_longlong(Eu);
            (void)Eb;
            // checkpoint rows this lane stores in this pass: row r (after
            // nuclide (r+1)*stride) exists iff (r+1)*stride <= ncomp and r < nck;
            // one compare per checkpoint instead of (ckon, mine, ncomp, nck)
            const int32_t ck_rows = (ckon && mine) ? min(nck, ncomp / kCkptStride) : 0;
            double* const ckp = MODE == 0 ? ckpt_of(S, s) : bout + n + i;
            for (int t = 0; t < nst; ++t, ++T) {
                const int d = (int)(T % LK_D);
                mbar_wait(&sh.full[d], (T / LK_D) & 1, 0x20000u | T);
                if (any && sh.sfast[d]) {
                    // every nuclide of the stage is fast (lk_fast): no per-nuclide
                    // meta word, clamp or branch -- the 8 folds' loads schedule freely
                    // brackets of all 8 nuclides first (independent broadcast loads,
                    // 2 bits each), so no record load waits on its own header load
                    uint32_t lis = 0;
#pragma unroll
                    for (int j = 0; j < LK_G; ++j) {
                        const longlong2 ab = sh.hdr[d][j];
#if EMC_LK_HDR_F64
                        lis |= ((uint32_t)(__longlong_as_double(ab.x) <= Eu) +
                                (uint32_t)(__longlong_as_double(ab.y) <= Eu)) << (2 * j);
#else
                        lis |= ((uint32_t)(ab.x <= Eb) + (uint32_t)(ab.y <= Eb)) << (2 * j);
#endif
                    }
#pragma unroll kLkFastUnroll
                    for (int j = 0; j < LK_G; ++j) {
                        const int k = t * LK_G + j;
                        const int32_t li = (int32_t)((lis >> (2 * j)) & 3u);
                        const IvRec* a = sh.iv[d][j] + li;
                        const double2 er = *reinterpret_cast<const double2*>(&a->E0);   // (E0, r)
                        const double e1 = a[1].E0;
                        const double2 tdt = *reinterpret_cast<const double2*>(&a->t0);
                        const double2 cdc = *reinterpret_cast<const double2*>(&a->c0);
                        const double2 fdf = *reinterpret_cast<const double2*>(&a->f0);
                        const double fr = div_by_rcp_safe(__dsub_rn(Eu, er.x), __dsub_rn(e1, er.x), er.y);
                        const double tt = __dadd_rn(tdt.x, __dmul_rn(fr, tdt.y));
                        const double cc = __dadd_rn(cdc.x, __dmul_rn(fr, cdc.y));
                        const double ff = __dadd_rn(fdf.x, __dmul_rn(fr, fdf.y));
                        const double2 dd =
                            DEN_ST ? *reinterpret_cast<const double2*>(sden + ((size_t)d * nmat + mu) * LK_DS + 2 * j)
                                   : *reinterpret_cast<const double2*>(&L.ddT[(int64_t)k * nmat + mu]);
                        st = __dadd_rn(st, __dmul_rn(dd.x, tt));
                        sc = __dadd_rn(sc, __dmul_rn(dd.x, cc));
                        sf = __dadd_rn(sf, __dmul_rn(dd.x, ff));
                        snf = __dadd_rn(snf, __dmul_rn(dd.y, ff));
                        if constexpr (kCkptStride < LK_G) {       // checkpoints inside the stage
                            if ((j + 1) % kCkptStride == 0) {
                                const int32_t row = (k + 1) / kCkptStride - 1;
                                if (row < ck_rows) ckp[(int64_t)row * cks] = st;
                            }
                        }
                    }
                } else if (any) {
#pragma unroll
                    for (int j = 0; j < LK_G; ++j) {
                        const int k = t * LK_G + j;
                        const uint32_t wd = sh.word[d][j];
                        const IvRec* W = sh.iv[d][j];
                        const double a1 = W[1].E0, a2 = W[2].E0;
                        double tt, cc, ff;
                        if (__builtin_expect(wd <= 4u, 1)) {
                            const int32_t li = min((int32_t)(a1 <= Eu) + (int32_t)(a2 <= Eu), (int32_t)wd - 2);
                            const double2 er = *reinterpret_cast<const double2*>(&W[li].E0);
                            const double e1 = W[li + 1].E0;
                            const IvRec& a = W[li];
                            const double fr = div_by_rcp_safe(__dsub_rn(Eu, er.x), __dsub_rn(e1, er.x), er.y);
                            tt = __dadd_rn(a.t0, __dmul_rn(fr, a.dt));
                            cc = __dadd_rn(a.c0, __dmul_rn(fr, a.dc));
                            ff = __dadd_rn(a.f0, __dmul_rn(fr, a.df));
                        } else {
                            lk_micro_slow(L, sh.meta[d][j], wd, W, a1, a2, bu, Eu, tt, cc, ff);
                        }
                        const double2 dd =
                            DEN_ST ? *reinterpret_cast<const double2*>(sden + ((size_t)d * nmat + mu) * LK_DS + 2 * j)
                                   : *reinterpret_cast<const double2*>(&L.ddT[(int64_t)k * nmat + mu]);
                        st = __dadd_rn(st, __dmul_rn(dd.x, tt));
                        sc = __dadd_rn(sc, __dmul_rn(dd.x, cc));
                        sf = __dadd_rn(sf, __dmul_rn(dd.x, ff));
                        snf = __dadd_rn(snf, __dmul_rn(dd.y, ff));
                        if constexpr (kCkptStride < LK_G) {       // checkpoints inside the stage
                            if ((j + 1) % kCkptStride == 0) {
                                const int32_t row = (k + 1) / kCkptStride - 1;
                                if (row < ck_rows) ckp[(int64_t)row * cks] = st;
                            }
                        }
                    }
                }
                if (any) {
                    constexpr int CKS = kCkptStride >= LK_G ? kCkptStride / LK_G : 1;
                    if (kCkptStride >= LK_G && (t + 1) % CKS == 0) {
                        const int32_t row = (t + 1) / CKS - 1;
                        if (row < ck_rows) ckp[(int64_t)row * cks] = st;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.empty[d]);
            }
            if (mine) {
                if (MODE == 0) {
                    P2 cc; cc.t = st; cc.c = sc; cc.f = sf; cc.nsf = snf;
                    (rdst ? rdst : S.ps)[s].c = cc;
                } else {
                    bout[i] = st + sc + sf + snf;
                }
                nl += (unsigned long long)(__ldg(L.mat_off + m + 1) - __ldg(L.mat_off + m));
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&P.dempty[slot]);
    }
    if (MODE == 0 && !producer) {
        warp_add_u64(cnt + CNT_INTERP_TRANSPORT, 4ull * nl);
        warp_add_u64(cnt + CNT_NUCLIDE_LOOKUPS, nl);
    }
}

// piped configurations: 0 = one 32-warp CTA per SM, 1 = two 16-warp CTAs per SM
// (their chunk boundaries overlap; needs the ring to fit twice in shared memory)
// 3 = 16 x 1 (128 registers), 4 = 24 x 1 (80), 5 = 12 x 2 (80)
constexpr int LK_NPCFG = 6;
constexpr int lk_pcfg_warps(int c) { return c == 1 || c == 3 ? 16 : c == 2 ? 10 : c == 4 ? 24 : c == 5 ? 12 : 32; }
constexpr int lk_pcfg_minb(int c) { return c == 1 || c == 5 ? 2 : c == 2 ? 3 : 1; }

template <int MODE, int PC>
inline cudaError_t lk_launch_piped_cfg(const DLib& L, const int32_t* q, int64_t n, DSlots S, int32_t fused,
                                       unsigned long long* cnt, const double* bE, const int32_t* bM, double* bout,
                                       int sm_count, size_t smem, cudaStream_t st, PState* rdst, const LkKeys& K)
{
    constexpr int NW = lk_pcfg_warps(PC), MB = lk_pcfg_minb(PC);
    constexpr int64_t chunk = (NW - 1) * 32;
    const unsigned nb = (unsigned)std::min<int64_t>((n + chunk - 1) / chunk, (int64_t)sm_count * MB);
    if (L.den_staged)
        k_lookup_piped<MODE, true, NW, MB><<<nb, NW * 32, smem, st>>>(q, (int32_t)n, L, S, fused, cnt, bE, bM, bout,
                                                                      rdst, K);
    else
        k_lookup_piped<MODE, false, NW, MB><<<nb, NW * 32, smem, st>>>(q, (int32_t)n, L, S, fused, cnt, bE, bM, bout,
                                                                       rdst, K);
    return cudaGetLastError();
}

template <int MODE>
inline cudaError_t lk_launch_piped(const DLib& L, const int32_t* q, int64_t n, DSlots S, int32_t fused,
                                   unsigned long long* cnt, const double* bE, const int32_t* bM, double* bout,
                                   int sm_count, size_t smem, cudaStream_t st, PState* rdst, const LkKeys& K,
                                   int pcfg = 0)
{
    switch (pcfg) {
#define EMC_PC(C) case C: return lk_launch_piped_cfg<MODE, C>(L, q, n, S, fused, cnt, bE, bM, bout, sm_count, smem, st, rdst, K);
    EMC_PC(1) EMC_PC(2) EMC_PC(3) EMC_PC(4) EMC_PC(5)
#undef EMC_PC
    default: break;
    }
    return lk_launch_piped_cfg<MODE, 0>(L, q, n, S, fused, cnt, bE, bM, bout, sm_count, smem, st, rdst, K);
}

}  // namespace emc

namespace emc {

// Launch configurations of the chunk-synchronous staged lookup (warps per CTA
// x CTAs per SM x particles per lane), used on the unsorted tail queues.
// EMC_LK_CFG selects one at run time (tuning); 2 (two 16-warp CTAs per SM,
// which the 3-stage ring lets fit) is the default.
constexpr int LK_NCFG = 4;
constexpr int lk_cfg_warps(int c) { return c == 1 ? 20 : c == 2 ? 16 : c == 3 ? 17 : 32; }
constexpr int lk_cfg_minb(int c) { return c == 1 || c == 2 ? 2 : 1; }
constexpr int lk_cfg_ppl(int c) { return c == 3 ? 2 : 1; }

template <int MODE, int CFG>
inline cudaError_t lk_launch_cfg(const DLib& L, const int32_t* q, int64_t n, DSlots S, int32_t fused,
                                 unsigned long long* cnt, const double* bE, const int32_t* bM, double* bout,
                                 int sm_count, size_t smem, cudaStream_t st, const unsigned int* nptr,
                                 PState* rdst)
{
    constexpr int NW = lk_cfg_warps(CFG), MB = lk_cfg_minb(CFG), PP = lk_cfg_ppl(CFG);
    constexpr int64_t chunk = (NW - 1) * 32 * PP;
    const unsigned nb = (unsigned)std::min<int64_t>((n + chunk - 1) / chunk, (int64_t)sm_count * MB);
    if (L.den_staged)
        k_lookup_staged<MODE, true, NW, MB, PP><<<nb, NW * 32, smem, st>>>(q, (int32_t)n, L, S, fused, cnt, bE, bM,
                                                                           bout, nptr, rdst);
    else
        k_lookup_staged<MODE, false, NW, MB, PP><<<nb, NW * 32, smem, st>>>(q, (int32_t)n, L, S, fused, cnt, bE, bM,
                                                                            bout, nptr, rdst);
    return cudaGetLastError();
}

template <int MODE>
inline cudaError_t lk_launch(int cfg, const DLib& L, const int32_t* q, int64_t n, DSlots S, int32_t fused,
                             unsigned long long* cnt, const double* bE, const int32_t* bM, double* bout, int sm_count,
                             size_t smem, cudaStream_t st, const unsigned int* nptr = nullptr,
                             PState* rdst = nullptr)
{
    switch (cfg) {
    case 1: return lk_launch_cfg<MODE, 1>(L, q, n, S, fused, cnt, bE, bM, bout, sm_count, smem, st, nptr, rdst);
    case 2: return lk_launch_cfg<MODE, 2>(L, q, n, S, fused, cnt, bE, bM, bout, sm_count, smem, st, nptr, rdst);
    case 3: return lk_launch_cfg<MODE, 3>(L, q, n, S, fused, cnt, bE, bM, bout, sm_count, smem, st, nptr, rdst);
    default: return lk_launch_cfg<MODE, 0>(L, q, n, S, fused, cnt, bE, bM, bout, sm_count, smem, st, nptr, rdst);
    }
}

template <int MODE, int CFG>
inline cudaError_t lk_set_smem_cfg(size_t smem)
{
    constexpr int NW = lk_cfg_warps(CFG), MB = lk_cfg_minb(CFG), PP = lk_cfg_ppl(CFG);
    cudaError_t e = cudaFuncSetAttribute(k_lookup_staged<MODE, true, NW, MB, PP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_lookup_staged<MODE, false, NW, MB, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
}

inline cudaError_t lk_set_smem(size_t smem)
{
    cudaError_t e;
    if ((e = lk_set_smem_cfg<0, 0>(smem)) || (e = lk_set_smem_cfg<0, 1>(smem)) || (e = lk_set_smem_cfg<0, 2>(smem)) ||
        (e = lk_set_smem_cfg<0, 3>(smem)) || (e = lk_set_smem_cfg<1, 0>(smem)) || (e = lk_set_smem_cfg<1, 1>(smem)) ||
        (e = lk_set_smem_cfg<1, 2>(smem)) || (e = lk_set_smem_cfg<1, 3>(smem)))
        return e;
    const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
#define EMC_PS(M, C) (e = cudaFuncSetAttribute(k_lookup_piped<M, true, lk_pcfg_warps(C), lk_pcfg_minb(C)>, a, (int)smem)) || \
                     (e = cudaFuncSetAttribute(k_lookup_piped<M, false, lk_pcfg_warps(C), lk_pcfg_minb(C)>, a, (int)smem))
    if (EMC_PS(0, 0) || EMC_PS(0, 1) || EMC_PS(0, 2) || EMC_PS(0, 3) || EMC_PS(0, 4) || EMC_PS(0, 5) ||
        EMC_PS(1, 0) || EMC_PS(1, 1) || EMC_PS(1, 2) || EMC_PS(1, 3) || EMC_PS(1, 4) || EMC_PS(1, 5))
        return e;
#undef EMC_PS
    return cudaSuccess;
}

}  // namespace emc
