// Test tool (not product code): evaluates the CUDA toolkit's own Philox4x32-10
// (curand_philox4x32_x.h, curand_Philox4x32_10) on the HOST, as an independent
// implementation the oracle's Philox is pinned against (DESIGN.md pin H0).
// stdin: lines "c0 c1 c2 c3 k0 k1" in hex; stdout: "x0 x1 x2 x3" in hex.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 r = curand_Philox4x32_10(make_uint4(c0, c1, c2, c3), make_uint2(k0, k1));
    std::printf("%08x %08x %08x %08x\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
