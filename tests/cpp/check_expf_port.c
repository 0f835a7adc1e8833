/* Exhaustive host check of the product's expf restatement
 * (paper_2509_01322_b200/csrc/libm_port.h) against this host's glibc expf,
 * the function the reference calls (tensor.hpp:183, graph.hpp:531).
 * argv[1] = stride over the 2^32 bit patterns (1 = exhaustive).
 * Prints "<checked> <mismatches> <first_bad_bits>". */
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <stdint.h>
#include "libm_port.h"

int main(int argc, char** argv) {
    uint64_t stride = argc > 1 ? strtoull(argv[1], 0, 10) : 1;
    uint64_t checked = 0, bad = 0;
    uint32_t first_bad = 0;
    for (uint64_t b = 0; b < (1ULL << 32); b += stride) {
        float x;
        uint32_t u = (uint32_t)b;
        memcpy(&x, &u, 4);
        float want = expf(x), got = scmoe_expf(x);
        uint32_t wu, gu;
        memcpy(&wu, &want, 4);
        memcpy(&gu, &got, 4);
        int same = (wu == gu) || (isnan(want) && isnan(got));
        if (!same) {
            if (!bad) first_bad = u;
            ++bad;
        }
        ++checked;
    }
    printf("%llu %llu 0x%08x\n", (unsigned long long)checked, (unsigned long long)bad, first_bad);
    return bad != 0;
}
