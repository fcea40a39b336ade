// Host-side known-answer source for the oracle's Philox4x32-10 pin: calls cuRAND's own
// curand_Philox4x32_10 (curand_philox4x32_x.h) on the HOST for a counter sweep and prints
// "c0 c1 c2 c3 k0 k1 -> o0 o1 o2 o3" lines.  A library routine, independent of oracle.c.
#include <cstdio>
#define QUALIFIERS static __forceinline__ __host__ __device__
#include <cuda_runtime.h>
#include <curand_philox4x32_x.h>
int main() {
  unsigned seeds[3][2] = {{0u, 0u}, {0xffffffffu, 0xffffffffu}, {0x243f6a88u, 0x85a308d3u}};
  for (int s = 0; s < 3; ++s)
    for (unsigned i = 0; i < 64; ++i) {
      uint4 c = make_uint4(i * 2654435761u, i ^ 0xdeadbeefu, (i << 24) | (2u << 16) | (i & 15), 0x80000000u | i);
      if (i == 0) c = make_uint4(0, 0, 0, 0);
      if (i == 1) c = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      uint2 k = make_uint2(seeds[s][0], seeds[s][1]);
      uint4 o = curand_Philox4x32_10(c, k);
      printf("%u %u %u %u %u %u %u %u %u %u\n", c.x, c.y, c.z, c.w, k.x, k.y, o.x, o.y, o.z, o.w);
    }
  return 0;
}
