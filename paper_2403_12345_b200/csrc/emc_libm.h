/* Bit-exact replicas of glibc 2.39 log / sin / cos (x86-64 FMA variants).
 *
 * Why: the reference transport kernels are numba @njit code whose log/sin/cos
 * calls (kernels.py:500-501 isotropic_from_u, :733 collision distance,
 * :919 fission-site energy, :971 source energy) lower to llvm.{log,sin,cos}.f64
 * and resolve to the process's glibc libm, i.e. the ifunc targets __log_fma /
 * __sin_fma / __cos_fma on any AVX2+FMA host.  glibc is not correctly rounded,
 * so CUDA's libdevice results differ from it in ~0.1% of calls, which would
 * make GPU histories diverge from the reference.  These routines follow the
 * FMA-variant machine code of glibc 2.39 (objdump of libm-2.39.a members
 * e_log-fma.o and s_sin-fma.o) operation for operation: every fused
 * multiply-add the compiler emitted is an explicit EMC_FMA, every other
 * operation is a separately rounded IEEE op, so host (gcc -ffp-contract=off)
 * and device (__dmul_rn/__dadd_rn/__fma_rn) evaluate the identical sequence.
 *
 * Tables come from the same libm (tools/gen_glibc_tables.py ->
 * emc_glibc_tables.h).  Domain covered exactly: log on all positive normal and
 * subnormal doubles, sin/cos for |x| < 105414350 (all transport arguments are
 * 2*pi*u in [0, 2*pi)).  Larger sin/cos arguments need glibc's __branred and
 * are not used anywhere on the transport path (they return NaN here).
 *
 * Licence note: derived from the GNU C Library 2.39 (sysdeps/ieee754/dbl-64
 * e_log.c / s_sin.c, FMA builds), which is Copyright (C) the Free Software
 * Foundation and contributors and licensed under the GNU Lesser General Public
 * License v2.1 or later.  This file and the generated emc_glibc_tables.h are
 * a derivative work of that code and are distributed under the same LGPL-2.1+
 * terms; the rest of this repository is not derived from glibc.
 *
 * Validated against the system libm by tests/test_libm_replica.py (host build,
 * ~10^8 samples of the transport argument distributions, 0 mismatches
 * required) and on the GPU by tests/test_gpu_parity.py.
 */
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define EMC_LIBM_FN __device__ __forceinline__
#define EMC_TABLE_QUAL __device__ const __align__(32)
/* table entries read together in one load (tables 32-byte aligned; on the
   device a lane's 2 / 4 entries are one 128- / 256-bit request instead of
   2 / 4 scattered 64-bit ones) */
#define EMC_TAB2(t, i, a, b) do { const double2 v_ = *reinterpret_cast<const double2*>(&(t)[i]); \
                                  (a) = v_.x; (b) = v_.y; } while (0)
#define EMC_TAB4(t, i, a, b, c, d) \
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(&(t)[i]))
#define EMC_FMA(a, b, c) __fma_rn((a), (b), (c))
#define EMC_MUL(a, b) __dmul_rn((a), (b))
#define EMC_ADD(a, b) __dadd_rn((a), (b))
#define EMC_SUB(a, b) __dsub_rn((a), (b))
#define EMC_AS_U64(x) ((uint64_t)__double_as_longlong(x))
#define EMC_AS_F64(u) __longlong_as_double((long long)(u))
#define EMC_FABS(x) fabs(x)
#else
#include <math.h>
#include <string.h>
#define EMC_LIBM_FN static inline
#define EMC_TABLE_QUAL const
#define EMC_TAB2(t, i, a, b) do { (a) = (t)[i]; (b) = (t)[(i) + 1]; } while (0)
#define EMC_TAB4(t, i, a, b, c, d) do { (a) = (t)[i]; (b) = (t)[(i) + 1]; (c) = (t)[(i) + 2]; (d) = (t)[(i) + 3]; } while (0)
#define EMC_FMA(a, b, c) fma((a), (b), (c))
#define EMC_MUL(a, b) ((a) * (b))
#define EMC_ADD(a, b) ((a) + (b))
#define EMC_SUB(a, b) ((a) - (b))
static inline uint64_t emc_as_u64_(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double emc_as_f64_(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
#define EMC_AS_U64(x) emc_as_u64_(x)
#define EMC_AS_F64(u) emc_as_f64_(u)
#define EMC_FABS(x) fabs(x)
#endif

#include "emc_glibc_tables.h"

/* ------------------------------------------------------------------ log --- */

EMC_LIBM_FN double emc_log(double x)
{
    uint64_t ix = EMC_AS_U64(x);
    /* |x - 1| < ~1/16: polynomial path (e_log-fma.o +0x100..0x1d2). */
    if (ix - 0x3fee000000000000ULL < 0x3090000000000ULL) {
        if (ix == 0x3ff0000000000000ULL) return 0.0;
        double r = EMC_SUB(x, 1.0);
        double p2 = EMC_FMA(r, EMC_LOG_B2, EMC_LOG_B1);
        double p5 = EMC_FMA(r, EMC_LOG_B5, EMC_LOG_B4);
        double r2 = EMC_MUL(r, r);
        double p8 = EMC_FMA(r, EMC_LOG_B8, EMC_LOG_B7);
        p2 = EMC_FMA(r2, EMC_LOG_B3, p2);
        p5 = EMC_FMA(r2, EMC_LOG_B6, p5);
        double r3 = EMC_MUL(r, r2);
        double q = EMC_FMA(r2, EMC_LOG_B9, p8);
        q = EMC_FMA(r3, EMC_LOG_B10, q);
        q = EMC_FMA(q, r3, p5);
        q = EMC_FMA(q, r3, p2);
        double rw = EMC_FMA(r, 0x1p27, r);          /* r + r*2^27 */
        double rhi = EMC_FMA(-0x1p27, r, rw);       /* (r + w) - w */
        double rhi2 = EMC_MUL(rhi, rhi);
        double rlo = EMC_SUB(r, rhi);
        double hi = EMC_FMA(rhi2, EMC_LOG_B0, r);
        double t8 = EMC_SUB(r, hi);
        double rpr = EMC_ADD(r, rhi);
        double lo = EMC_FMA(rhi2, EMC_LOG_B0, t8);
        double t2 = EMC_MUL(EMC_LOG_B0, rlo);
        lo = EMC_FMA(t2, rpr, lo);
        double y = EMC_FMA(q, r3, lo);
        return EMC_ADD(hi, y);
    }
    uint32_t top = (uint32_t)(ix >> 48);
    if (top - 0x0010u > 0x7fdfu) {
        /* x < 0x1p-1022, negative, inf or nan */
        if ((ix << 1) == 0) return -1.0 / 0.0;            /* log(+-0) = -inf */
        if (ix == 0x7ff0000000000000ULL) return x;         /* log(inf) = inf */
        if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return (x - x) / (x - x);
        /* subnormal: normalise (x * 2^52, exponent - 52) */
        ix = EMC_AS_U64(EMC_MUL(x, 0x1p52));
        ix -= 52ULL << 52;
    }
    /* table path (e_log-fma.o +0x3f..0xfb) */
    uint64_t tmp = ix - 0x3fe6000000000000ULL;
    int i = (int)((tmp >> 45) & 0x7f);
    int32_t k = (int32_t)((int64_t)tmp >> 52);
    uint64_t iz = ix - (tmp & 0xfff0000000000000ULL);
    double invc, logc;
    EMC_TAB2(emc_log_tab, 2 * i, invc, logc);
    double kd = (double)k;
    double z = EMC_AS_F64(iz);
    double w = EMC_FMA(kd, EMC_LOG_LN2HI, logc);
    double r = EMC_FMA(z, invc, -1.0);
    double p12 = EMC_FMA(r, EMC_LOG_A2, EMC_LOG_A1);
    double hi = EMC_ADD(r, w);
    double r2 = EMC_MUL(r, r);
    double lo = EMC_ADD(EMC_SUB(w, hi), r);
    lo = EMC_FMA(kd, EMC_LOG_LN2LO, lo);
    double r3 = EMC_MUL(r, r2);
    double p34 = EMC_FMA(r, EMC_LOG_A4, EMC_LOG_A3);
    lo = EMC_FMA(r2, EMC_LOG_A0, lo);
    double p = EMC_FMA(p34, r2, p12);
    double y = EMC_FMA(r3, p, lo);
    return EMC_ADD(y, hi);
}

/* -------------------------------------------------------------- sin/cos --- */
/* s_sin.c constants (EMC_SC_*) come from s_sin-fma.o .rodata.cst8 via emc_glibc_tables.h */

EMC_LIBM_FN double emc_copysign_(double mag, double sgn)
{
    uint64_t m = EMC_AS_U64(mag) & 0x7fffffffffffffffULL;
    uint64_t s = EMC_AS_U64(sgn) & 0x8000000000000000ULL;
    return EMC_AS_F64(m | s);
}

/* TAYLOR_SIN(a*a, a, da) */
EMC_LIBM_FN double emc_taylor_sin_(double a, double da)
{
    double xx = EMC_MUL(a, a);
    double p = EMC_FMA(xx, EMC_SC_S5, EMC_SC_S4);
    p = EMC_FMA(xx, p, EMC_SC_S3);
    p = EMC_FMA(xx, p, EMC_SC_S2);
    p = EMC_FMA(xx, p, EMC_SC_S1);
    double hda = EMC_MUL(da, 0.5);
    double t = EMC_FMA(p, a, -hda);
    t = EMC_FMA(xx, t, da);
    return EMC_ADD(t, a);
}

/* do_sin for |x| >= 0.126: table + correction, copysign(x) */
EMC_LIBM_FN double emc_do_sin_tab_(double x, double dx)
{
    if (x <= 0.0) dx = -dx;
    double ax = EMC_FABS(x);
    double u = EMC_ADD(ax, EMC_SC_BIG);
    int k = (int)(uint32_t)EMC_AS_U64(u) << 2;
    double xr = EMC_SUB(ax, EMC_SUB(u, EMC_SC_BIG));
    double sn, ssn, cs, ccs;
    EMC_TAB4(emc_sincostab, k, sn, ssn, cs, ccs);
    double xx = EMC_MUL(xr, xr);
    double ps = EMC_FMA(xx, EMC_SC_SN5, EMC_SC_SN3);
    double s = EMC_FMA(EMC_MUL(xr, xx), ps, dx);
    double pc = EMC_FMA(xx, EMC_SC_CS6, EMC_SC_CS4);
    pc = EMC_FMA(xx, pc, EMC_SC_CS2);
    s = EMC_ADD(xr, s);
    double c = EMC_FMA(xr, dx, EMC_MUL(xx, pc));
    double t = EMC_FMA(s, ccs, ssn);
    t = EMC_FMA(-c, sn, t);
    t = EMC_FMA(s, cs, t);
    return emc_copysign_(EMC_ADD(sn, t), x);
}

EMC_LIBM_FN double emc_do_sin_(double x, double dx)
{
    if (EMC_FABS(x) < EMC_SC_TAYLOR_MAX) return emc_taylor_sin_(x, dx);
    return emc_do_sin_tab_(x, dx);
}

EMC_LIBM_FN double emc_do_cos_(double x, double dx)
{
    if (x < 0.0) dx = -dx;
    double ax = EMC_FABS(x);
    double u = EMC_ADD(ax, EMC_SC_BIG);
    int k = (int)(uint32_t)EMC_AS_U64(u) << 2;
    double xr = EMC_ADD(EMC_SUB(ax, EMC_SUB(u, EMC_SC_BIG)), dx);
    double sn, ssn, cs, ccs;
    EMC_TAB4(emc_sincostab, k, sn, ssn, cs, ccs);
    double xx = EMC_MUL(xr, xr);
    double ps = EMC_FMA(xx, EMC_SC_SN5, EMC_SC_SN3);
    double s = EMC_FMA(EMC_MUL(xr, xx), ps, xr);
    double pc = EMC_FMA(xx, EMC_SC_CS6, EMC_SC_CS4);
    pc = EMC_FMA(xx, pc, EMC_SC_CS2);
    double c = EMC_MUL(xx, pc);
    double t = EMC_FMA(-s, ssn, ccs);
    t = EMC_FMA(-c, cs, t);
    t = EMC_FMA(-s, sn, t);
    return EMC_ADD(cs, t);
}

/* reduce_sincos: x -> (a, da, quadrant) for 2.426265 <= |x| < 105414350 */
EMC_LIBM_FN int emc_reduce_sincos_(double x, double *a, double *da)
{
    double t = EMC_FMA(x, EMC_SC_HPINV, EMC_SC_TOINT);
    double xn = EMC_SUB(t, EMC_SC_TOINT);
    int n = (int)((uint32_t)EMC_AS_U64(t) & 3u);
    double y = EMC_FMA(-xn, EMC_SC_MP1, x);
    y = EMC_FMA(-xn, EMC_SC_MP2, y);
    double t2 = EMC_FMA(-xn, EMC_SC_PP3, y);
    double db = EMC_FMA(-xn, EMC_SC_PP3, EMC_SUB(y, t2));
    double b = EMC_FMA(-xn, EMC_SC_PP4, t2);
    double e = EMC_FMA(-xn, EMC_SC_PP4, EMC_SUB(t2, b));
    *a = b;
    *da = EMC_ADD(db, e);
    return n;
}

EMC_LIBM_FN double emc_sin(double x)
{
    uint32_t k = (uint32_t)(EMC_AS_U64(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e500000u) return x;
    if (k < 0x3feb6000u) return emc_do_sin_(x, 0.0);
    if (k < 0x400368fdu) {
        double t = EMC_SUB(EMC_SC_HP0, EMC_FABS(x));
        return emc_copysign_(emc_do_cos_(t, EMC_SC_HP1), x);
    }
    if (k < 0x419921fbu) {
        double a, da;
        int n = emc_reduce_sincos_(x, &a, &da);
        double r = (n & 1) ? emc_do_cos_(a, da) : emc_do_sin_(a, da);
        return (n & 2) ? -r : r;
    }
    return (x - x) / (x - x);   /* huge / inf / nan: not on the transport path */
}

EMC_LIBM_FN double emc_cos(double x)
{
    uint32_t k = (uint32_t)(EMC_AS_U64(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e400000u) return 1.0;
    if (k < 0x3feb6000u) return emc_do_cos_(x, 0.0);
    if (k < 0x400368fdu) {
        double y = EMC_SUB(EMC_SC_HP0, EMC_FABS(x));
        double a = EMC_ADD(y, EMC_SC_HP1);
        double da = EMC_ADD(EMC_SUB(y, a), EMC_SC_HP1);
        return emc_do_sin_(a, da);
    }
    if (k < 0x419921fbu) {
        double a, da;
        int n = emc_reduce_sincos_(x, &a, &da) + 1;
        double r = (n & 1) ? emc_do_cos_(a, da) : emc_do_sin_(a, da);
        return (n & 2) ? -r : r;
    }
    return (x - x) / (x - x);
}
