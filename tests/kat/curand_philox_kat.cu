// Test-only known-answer generator: curand's own Philox4x32-10, compiled for
// the HOST by overriding QUALIFIERS.  Reads lines "c0 c1 c2 c3 k0 k1" (hex)
// on stdin and prints the four output words (hex) per line.  Used by
// tests/test_oracle_philox.py to pin oracle/philox.py against an independent
// implementation; never linked into the product.
#define QUALIFIERS static __host__ __device__ __forceinline__
#include <curand_philox4x32_x.h>
#include <cstdio>

int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = make_uint4(c0, c1, c2, c3);
    uint2 k = make_uint2(k0, k1);
    uint4 r = curand_Philox4x32_10(c, k);
    std::printf("%08x %08x %08x %08x\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
