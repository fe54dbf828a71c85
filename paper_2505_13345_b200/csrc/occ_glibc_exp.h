// occ_glibc_exp.h — glibc's double exp, bit for bit, on the device (and host).
//
// The reference's softmax calls std::exp (routing.cpp:44), i.e. glibc's libm
// exp (sysdeps/ieee754/dbl-64/e_exp.c, the optimized-routines algorithm,
// glibc >= 2.28).  On x86-64 with FMA (every host this build targets) the
// ifunc picks the FMA compilation of that source, whose contractions are
// replicated here operation for operation (read off `objdump -d` of this
// image's libm __exp_fma; constants from __exp_data, table from
// gen_exp_table.py):
//
//   kd  = fma(x, N/ln2, 0x1.8p52);  ki = bits(kd);  kd -= 0x1.8p52
//   r   = fma(kd, -ln2hi/N, x);  r = fma(kd, -ln2lo/N, r)
//   tmp = fma(r2 * r2, fma(r, C5, C4), fma(fma(r, C3, C2), r2, r + tail))
//   exp = fma(scale, tmp, scale),  scale = 2^(ki/N) from the table
//
// plus the tiny / huge / subnormal special cases (e_exp.c specialcase(),
// which multiplies and adds separately).  Every operation is an explicit
// round-to-nearest intrinsic on the device, so nvcc cannot contract or
// reassociate; host builds must use -ffp-contract=off.  Checked against
// libm on 2^26 random arguments per range, incl. all special cases
// (tests/test_exp_port.py), and end to end by the bit-exact gate_scores tests.
#pragma once
#include <stdint.h>

#include "occ_exp_table.h"

#ifdef __CUDACC__
#define OCC_HD __host__ __device__ __forceinline__
#else
#define OCC_HD inline
#include <math.h>
#include <string.h>
#endif

namespace occ {
namespace glibc_exp {

#ifdef __CUDACC__
static __device__ const uint64_t kTabDev[256] = OCC_EXP_TABLE_INIT;
#endif
static const uint64_t kTabHost[256] = OCC_EXP_TABLE_INIT;

OCC_HD uint64_t tab(int i) {
#ifdef __CUDA_ARCH__
    return __ldg(reinterpret_cast<const unsigned long long*>(kTabDev) + i);
#else
    return kTabHost[i];
#endif
}

OCC_HD double as_double(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double d;
    memcpy(&d, &u, 8);
    return d;
#endif
}
OCC_HD uint64_t as_u64(double d) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
#endif
}

#ifdef __CUDA_ARCH__
OCC_HD double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
OCC_HD double add_(double a, double b) { return __dadd_rn(a, b); }
OCC_HD double sub_(double a, double b) { return __dsub_rn(a, b); }
OCC_HD double mul_(double a, double b) { return __dmul_rn(a, b); }
#else
OCC_HD double fma_(double a, double b, double c) { return fma(a, b, c); }
OCC_HD double add_(double a, double b) { return a + b; }
OCC_HD double sub_(double a, double b) { return a - b; }
OCC_HD double mul_(double a, double b) { return a * b; }
#endif

// __exp_data (math_config.h): N = 128 table entries.
constexpr double kInvLn2N = 0x1.71547652b82fep7;
constexpr double kShift = 0x1.8p52;
constexpr double kNegLn2hiN = -0x1.62e42fefa0000p-8;
constexpr double kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
constexpr double kC2 = 0x1.ffffffffffdbdp-2;
constexpr double kC3 = 0x1.555555555543cp-3;
constexpr double kC4 = 0x1.55555cf172b91p-5;
constexpr double kC5 = 0x1.1111167a4d017p-7;

// e_exp.c specialcase(): |x| large enough that scale over/underflows.
OCC_HD double special(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000u) == 0) {  // k > 0: scale's exponent overflowed by <= 460
        sbits -= 1009ull << 52;
        const double scale = as_double(sbits);
        return mul_(fma_(scale, tmp, scale), 0x1p1009);
    }
    sbits += 1022ull << 52;  // k < 0: careful subnormal rounding
    const double scale = as_double(sbits);
    const double st = mul_(tmp, scale);
    double y = add_(scale, st);
    if (y < 1.0) {
        const double hi = add_(y, 1.0);
        double lo = add_(sub_(scale, y), st);
        lo = add_(add_(sub_(1.0, hi), y), lo);
        y = sub_(add_(lo, hi), 1.0);
        if (y == 0.0) return 0.0;
    }
    return mul_(y, 0x1p-1022);
}

OCC_HD double exp(double x) {
    const uint64_t ix = as_u64(x);
    uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {          // |x| < 2^-54 or |x| >= 512
        if ((int32_t)(abstop - 0x3c9u) < 0)   // tiny: avoid spurious underflow
            return add_(1.0, x);
        if (abstop >= 0x409) {                // |x| >= 1024
            if (ix == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ff) return add_(1.0, x);  // inf / nan
            if (ix >> 63) return mul_(0x1p-767, 0x1p-767);   // __math_uflow(0)
            return mul_(0x1p769, 0x1p769);                  // __math_oflow(0)
        }
        abstop = 0;  // large x: special-cased below
    }
    double kd = fma_(x, kInvLn2N, kShift);
    const uint64_t ki = as_u64(kd);
    kd = sub_(kd, kShift);
    double r = fma_(kd, kNegLn2hiN, x);
    r = fma_(kd, kNegLn2loN, r);
    const int idx = 2 * (int)(ki % 128);
    const uint64_t top = ki << 45;
    const double tail = as_double(tab(idx));
    const uint64_t sbits = tab(idx + 1) + top;
    const double r2 = mul_(r, r);
    const double p23 = fma_(r, kC3, kC2);
    const double tr = add_(r, tail);
    const double p45 = fma_(r, kC5, kC4);
    double tmp = fma_(p23, r2, tr);
    tmp = fma_(mul_(r2, r2), p45, tmp);
    if (abstop == 0) return special(tmp, sbits, ki);
    const double scale = as_double(sbits);
    return fma_(scale, tmp, scale);
}

}  // namespace glibc_exp
}  // namespace occ
