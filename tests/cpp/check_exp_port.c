/* Host check of the product's glibc-exp (double) restatement
 * (paper_2509_01322_b200/csrc/libm_port.h) against this host's glibc exp,
 * the function the reference's RouterState<double> softmax calls
 * (tensor.hpp:183).  argv[1] = number of xorshift samples: a third over
 * [-750, 750] (incl. the subnormal/overflow special cases), a third over the
 * softmax domain [-30, 10], a third tiny negatives; plus fixed edge values.
 * Prints "<checked> <mismatches> <first_bad_bits>". */
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <stdint.h>
#include "libm_port.h"

static int same(double a, double b) {
    uint64_t ua, ub;
    memcpy(&ua, &a, 8);
    memcpy(&ub, &b, 8);
    return ua == ub || (isnan(a) && isnan(b));
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 10000000;
    const double edges[] = {0.0, -0.0, 1.0, -1.0, 709.78, 709.79, 710.0, -708.39, -708.4, -745.13,
                            -745.14, -746.0, 0x1p-54, -0x1p-54, 0x1p-60, 512.0, -512.0, 1024.0,
                            -1024.0, INFINITY, -INFINITY, NAN};
    uint64_t checked = 0, bad = 0, first = 0, s = 0x9E3779B97F4A7C15ull;
    for (size_t i = 0; i < sizeof(edges) / sizeof(edges[0]); ++i, ++checked)
        if (!same(exp(edges[i]), scmoe_exp(edges[i]))) {
            if (!bad) memcpy(&first, &edges[i], 8);
            ++bad;
        }
    for (uint64_t i = 0; i < n; ++i, ++checked) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        const double u = (double)(s >> 11) * 0x1p-53;
        const double x = i % 3 == 0 ? u * 1500.0 - 750.0 : i % 3 == 1 ? u * 40.0 - 30.0 : -u * 1e-3;
        if (!same(exp(x), scmoe_exp(x))) {
            if (!bad) memcpy(&first, &x, 8);
            ++bad;
        }
    }
    printf("%llu %llu %llx\n", (unsigned long long)checked, (unsigned long long)bad,
           (unsigned long long)first);
    return 0;
}
