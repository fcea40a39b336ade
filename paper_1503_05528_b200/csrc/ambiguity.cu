// ambiguity.cu — App. B, Table 2: Monte-Carlo probability that
// a random patch V is closer (SSD) to a random reference patch W than the constant patch Z = mu,
// components i.i.d. N(mu, sigma^2).  The paper's direct simulation, one trial per thread-iteration:
// 2N normals from Philox4x32-10 (counter = (trial lo, trial hi, 4 << 16 | k, 0)) by fp64 Box-Muller,
// W_c = normal 2c, V_c = normal 2c + 1; hit iff sum (W - V)^2 < sum (W - mu)^2.  Hit counts are
// exact integers (int64 atomics), so ranks can split trial ranges and all-reduce.
#include "common.cuh"

namespace vinp {

__global__ void __launch_bounds__(256) k_ambiguity(int N, double sigma, uint64_t seed, uint64_t trial0,
                                                   uint64_t n_trials, unsigned long long* __restrict__ hits) {
  unsigned long long h = 0;
  const double two_pi = 6.283185307179586476925286766559;
  for (uint64_t tr = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; tr < n_trials;
       tr += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t t = trial0 + tr;
    double a = 0.0, b = 0.0, w = 0.0;
    int nn = 2 * N;
    for (int k = 0; k < (nn + 3) / 4; ++k) {
      uint4 u = philox(make_uint4((uint32_t)t, (uint32_t)(t >> 32), (4u << 16) | (uint32_t)k, 0u),
                       (uint32_t)seed, (uint32_t)(seed >> 32));
      double r1 = sqrt(-2.0 * log(((double)u.x + 0.5) / 4294967296.0));
      double r2 = sqrt(-2.0 * log(((double)u.z + 0.5) / 4294967296.0));
      double s1, c1, s2, c2;
      sincos(two_pi * ((double)u.y / 4294967296.0), &s1, &c1);
      sincos(two_pi * ((double)u.w / 4294967296.0), &s2, &c2);
      double z[4] = {r1 * c1, r1 * s1, r2 * c2, r2 * s2};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int idx = 4 * k + j;
        if (idx < nn) {
          if ((idx & 1) == 0) {
            w = sigma * z[j];
          } else {
            double v = sigma * z[j];
            a += (w - v) * (w - v);
            b += w * w;
          }
        }
      }
    }
    h += (a < b);
  }
  h = __reduce_add_sync(kFull, (unsigned)h);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(hits, h);
}

}  // namespace vinp

using namespace vinp;

extern "C" {

vinp_status vinp_patch_ambiguity(int N, double sigma, uint64_t seed, uint64_t trial0, uint64_t n_trials,
                                 unsigned long long* hits, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(N >= 1 && N <= 4096 && sigma > 0 && hits, "vinp_patch_ambiguity: bad arguments");
  if (n_trials == 0) return VINP_OK;
  uint64_t blocks = std::min<uint64_t>((n_trials + 255) / 256, 148ull * 16);
  k_ambiguity<<<(unsigned)blocks, 256, 0, S(stream)>>>(N, sigma, seed, trial0, n_trials, hits);
  count_launch();
  return check_launch("vinp_patch_ambiguity");
}

}  // extern "C"
