// Pin for the oracle's Philox4x32-10: cuRAND's own raw block function
// (curand_philox4x32_x.h, curand_Philox4x32_10) compiled for the HOST.
// Reads "c0 c1 c2 c3 k0 k1" lines (hex) on stdin, prints the 4 output words.
#include <cstdio>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main() {
    unsigned c0, c1, c2, c3, k0, k1;
    while (std::scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
        uint4 c = {c0, c1, c2, c3};
        uint2 k = {k0, k1};
        uint4 r = curand_Philox4x32_10(c, k);
        std::printf("%08x %08x %08x %08x\n", r.x, r.y, r.z, r.w);
    }
    return 0;
}
