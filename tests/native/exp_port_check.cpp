// Host check of the device exp port (paper_2505_13345_b200/csrc/occ_glibc_exp.h)
// against this machine's libm exp, bit for bit.  Built with -ffp-contract=off
// by tests/test_exp_port.py.  Usage: exp_port_check <samples_per_range> <seed>
// Prints "ranges=R checked=N mismatches=M" and the first few mismatches.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "occ_glibc_exp.h"

static uint64_t bits(double d) { uint64_t u; std::memcpy(&u, &d, 8); return u; }
static double from(uint64_t u) { double d; std::memcpy(&d, &u, 8); return d; }

int main(int argc, char** argv) {
    const long per = argc > 1 ? atol(argv[1]) : 1000000;
    std::mt19937_64 g(argc > 2 ? strtoull(argv[2], nullptr, 10) : 1);
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    struct Range { double lo, hi; } ranges[] = {
        {-60.0, 0.0},      // softmax arguments x - max of realistic logits
        {-1.0, 1.0},       {-745.2, -700.0},  // subnormal results (specialcase k < 0)
        {700.0, 709.8},    // specialcase k > 0
        {-1100.0, 1100.0}, // over / underflow, |x| >= 1024
        {-1e-15, 1e-15},   // tiny
    };
    long checked = 0, bad = 0;
    auto check = [&](double x) {
        const double want = std::exp(x), got = occ::glibc_exp::exp(x);
        ++checked;
        if (bits(want) != bits(got) && !(std::isnan(want) && std::isnan(got))) {
            if (bad < 8) std::printf("mismatch x=%a libm=%a port=%a\n", x, want, got);
            ++bad;
        }
    };
    for (const Range& r : ranges)
        for (long i = 0; i < per; ++i) check(r.lo + (r.hi - r.lo) * u01(g));
    for (long i = 0; i < per; ++i) check(from(g()));  // arbitrary bit patterns
    const double specials[] = {0.0, -0.0, INFINITY, -INFINITY, NAN, 0x1p-54, -0x1p-54, 0x1p-55, 512.0, -512.0,
                               1024.0, -1024.0, 709.782712893384, -745.1332191019411, -708.3964185322641,
                               0x1.62e42fefa39efp+9, -0x1.74910d52d3051p+9, 4.9406564584124654e-324};
    for (double x : specials) check(x);
    std::printf("ranges=%d checked=%ld mismatches=%ld\n", (int)(sizeof(ranges) / sizeof(ranges[0])) + 1, checked, bad);
    return bad != 0;
}
