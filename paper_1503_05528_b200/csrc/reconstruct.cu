// reconstruct.cu — patch-vote reconstruction (a9/a10: Eqs. 4-6, 11, 13), commit of the u8
// working copy, the stopping-rule change (a11) and the Eq. 1 energy diagnostic.
//
// One warp per hole pixel p, gathering its <= 125 contributors q in N_p (lane l owns q = p + off_v
// for v = l + 32i): each lane reads slot[q], the NNF entry of q and the proposed value
// u(p + phi(q)) = vox[src_q - off_v] — a per-target-pixel gather, no atomics (north_star (c)).
// sigma_p^2 is selected exactly as the ceil(0.75 m)-th smallest key d^2 = D/n (the key is the
// fp64 D/n, which orders distinct rationals with n <= 125 exactly) by a bitwise rank search with
// one REDUX.SUM per bit: on the high 32 key bits from the first bit where the warp's keys differ,
// and on the low 32 bits only if the selected high half is shared by unequal keys.  Weights are
// round(exp(-a) 2^36) so that the sums are exact integers, independent of reduction order (R26);
// they are summed as two 23-bit halves with REDUX.SUM.
#include "common.cuh"

namespace vinp {

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }
#ifndef VINP_REC_WPB
#define VINP_REC_WPB 8
#endif
constexpr int kWPB = VINP_REC_WPB;

__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(kFull, (uint32_t)v, m), hi = __shfl_xor_sync(kFull, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v += (int64_t)shfl_xor64((uint64_t)v, m);
  return v;
}
// exact warp sum of non-negative values < 2^46 (two 23-bit halves, each < 2^28 summed)
__device__ __forceinline__ int64_t warp_sum46(int64_t v) {
  uint32_t lo = (uint32_t)(v & 0x7fffff), hi = (uint32_t)(v >> 23);
  lo = __reduce_add_sync(kFull, lo);
  hi = __reduce_add_sync(kFull, hi);
  return ((int64_t)hi << 23) + lo;
}
__device__ __forceinline__ uint64_t warp_min64(uint64_t v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v = min(v, shfl_xor64(v, m));
  return v;
}

__device__ __forceinline__ uint8_t round_u8(float x) {
  return (uint8_t)floor((double)x + 0.5);
}

#ifndef VINP_REC_PREFETCH
#define VINP_REC_PREFETCH 0  // 1: stage A (slot gathers) of the next hole issued before this hole's arithmetic (A/B: 17.5 vs 17.5-17.9 ms, 44 B of spills at 64 registers; 85 registers: 18.9 ms)
#endif
#ifndef VINP_REC_CHUNKED
#define VINP_REC_CHUNKED 1  // A/B at c5 level 1: strided persistent warps 15.2 ms (2 waves) / 14.2 (64); contiguous chunks 16.9 (2 waves: imbalance) / 13.3 (32) / 13.2 (64) / 13.3 (256) / 14.7 (1024)
#endif
#ifndef VINP_REC_WAVES
#define VINP_REC_WAVES 64
#endif
#ifndef VINP_REC_MINB
#define VINP_REC_MINB 4
#endif

// 2^(j/128) = hi (1 + tail), j = 0..127 (tools/gen_exp_table.py); staged in shared memory per block
__device__ const double2 kExpTab[128] = {
#include "exp_tab.inc"
};

// round(2^36 exp(-a)), a >= 0, the weight of Eq. 5 in the fixed point of R31.  exp by the usual
// table-driven reduction: -a = (128 k + j) ln2/128 + r, |r| <= ln2/256, exp(-a) = 2^k 2^(j/128) e^r
// with a degree-5 polynomial for e^r - 1 (|error| < 2^-60) and a (hi, tail) table entry, about
// 0.51 ulp; 2^36 is folded into the exponent and the rounding to an integer is the 1.5 * 2^52
// shift (round half to even, as llrint).  Against glibc's exp followed by llrint: 2 of 6.5e8 weights
// differ, by one unit of 2^-36 (host prototype of the same arithmetic).
__device__ __forceinline__ int64_t weight36(double a, const double2* __restrict__ tab) {
  const double InvLn2N = 0x1.71547652b82fep+7, Shift = 0x1.8p52;
  const double Ln2hiN = 0x1.62e42fefa0000p-8, Ln2loN = 0x1.cf79abc9e3b3ap-47;
  const double x = -fmin(a, 64.0);  // 2^36 exp(-64) < 2^-56 rounds to 0 like every larger a
  const double t = __fma_rn(x, InvLn2N, Shift);
  const int ki = __double2loint(t);
  const double kd = __dadd_rn(t, -Shift);
  double r = __fma_rn(kd, -Ln2hiN, x);
  r = __fma_rn(kd, -Ln2loN, r);
  const double r2 = __dmul_rn(r, r);
  const double pa = __fma_rn(r, 1.0 / 6, 0.5), pb = __fma_rn(r, 1.0 / 120, 1.0 / 24);
  const double2 T = tab[ki & 127];
  double tmp = __dadd_rn(T.y, r);
  tmp = __fma_rn(r2, pa, tmp);
  tmp = __fma_rn(__dmul_rn(r2, r2), pb, tmp);
  const double sc = __hiloint2double(__double2hiint(T.x) + (((ki >> 7) + 36) << 20), __double2loint(T.x));
  const double u = __dadd_rn(__fma_rn(sc, tmp, sc), Shift);
  return ((int64_t)(__double2hiint(u) - 0x43380000) << 32) | (uint32_t)__double2loint(u);
}

// The r-th smallest (1-based) of the warp's valid 32-bit keys k[0..3] per lane (invalid = ~0, valid
// < 2^31; m >= r valid keys in the warp): bitwise rank search from the first bit where the keys
// differ, one REDUX.SUM per bit, ended as soon as a round's count c = #{keys <= T} is r or r - 1:
// the wanted key is then the largest key <= T or the smallest key > T (one REDUX.MAX / MIN) — a
// few rounds instead of one per bit.
__device__ __forceinline__ uint32_t select_rank32(const uint32_t (&k)[4], unsigned valid, uint32_t r, uint32_t m) {
  const uint32_t kmin = __reduce_min_sync(kFull, min(min(k[0], k[1]), min(k[2], k[3])));
  if (r == 1) return kmin;
  if (kmin == 0) {  // sigma_p = 0 is common (exact copies): r or more zero keys settle it at once
    uint32_t c = (k[0] == 0) + (k[1] == 0) + (k[2] == 0) + (k[3] == 0);
    if (__reduce_add_sync(kFull, c) >= r) return 0;
  }
  const uint32_t kmax = __reduce_max_sync(kFull, max(max((valid & 1) ? k[0] : 0u, (valid & 2) ? k[1] : 0u),
                                                     max((valid & 4) ? k[2] : 0u, (valid & 8) ? k[3] : 0u)));
  if (r == m) return kmax;
  const uint32_t x = kmax ^ kmin;
  if (x == 0) return kmin;  // all keys equal
  uint32_t ans = kmin & ~(0xffffffffu >> __clz(x));
  for (uint32_t b = 0x80000000u >> __clz(x); b; b >>= 1) {
    const uint32_t T = ans | (b - 1);
    uint32_t c = (k[0] <= T) + (k[1] <= T) + (k[2] <= T) + (k[3] <= T);
    c = __reduce_add_sync(kFull, c);
    if (c == r) {  // the wanted key is the largest key <= T
      uint32_t v = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) v = max(v, k[i] <= T ? k[i] : 0u);
      return __reduce_max_sync(kFull, v);
    }
    if (c + 1 == r) {  // ... or the smallest key > T (invalid keys are ~0, above every valid one)
      uint32_t v = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < 4; ++i) v = min(v, k[i] > T ? k[i] : 0xffffffffu);
      return __reduce_min_sync(kFull, v);
    }
    if (c < r) ans |= b;
  }
  return ans;
}

struct ReconArgs {
  Geo g;
  uint64_t* vox;
  const uint8_t* layer;
  const int32_t* slot;
  const int32_t* holes;
  const uint64_t* e;
  const uint8_t* n;
};

// Per-lane contributor geometry, the same for every hole: contributor v = lane + 32 i of N_p is the
// patch voxel (vdx, vdy, vdt), at linear offset off from p.
struct LaneVox {
  int off[4];
  int8_t dx[4], dy[4], dt[4];
  bool real[4];  // v < 125
};

// Stage A of a hole: its voxel, which of the lane's four contributors exist, and their slot loads.
// Issued one hole ahead by the persistent loop (VINP_REC_PREFETCH), so that two of the four
// dependent gather rounds of a hole overlap the arithmetic of the previous one.
struct HoleA {
  int h, p;
  int sl[4];
  unsigned cand;  // bit i: contributor i is a voxel of N_p in Omega (and in an earlier layer)
};

__device__ __forceinline__ HoleA recon_stage_a(const ReconArgs& a, const LaneVox& LV, int layer_j, int h) {
  HoleA A;
  A.h = h;
  const int p = a.holes[h];
  A.p = p;
  int px, py, pt;
  decode(a.g, p, px, py, pt);
  const int* off = LV.off;
  bool cand[4];
  // interior hole (the usual case): every voxel of N_p is in the volume, no per-voxel test
  const bool interior = px >= 2 && px < a.g.W - 2 && py >= 2 && py < a.g.H - 2 && pt >= 2 && pt < a.g.T - 2;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    cand[i] = LV.real[i] && (interior || inside(a.g, px + LV.dx[i], py + LV.dy[i], pt + LV.dt[i]));
  if (layer_j >= 0) {
    const bool mine = a.layer[p] == layer_j;  // other layers' holes: no contributor, nothing written
#pragma unroll
    for (int i = 0; i < 4; ++i) cand[i] = cand[i] && mine && a.layer[p + (cand[i] ? off[i] : 0)] < layer_j;
  }
  A.cand = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    A.sl[i] = __ldg(a.slot + p + (cand[i] ? off[i] : 0));
    A.cand |= (unsigned)cand[i] << i;
  }
  return A;
}

__device__ __forceinline__ void recon_hole(const ReconArgs& a, const LaneVox& LV, int lane, int mode, int layer_j,
                                           const HoleA& A, float* __restrict__ out_rgb, float* __restrict__ out_tex,
                                           int commit, const double2* __restrict__ tab) {
  const int h = A.h, p = A.p;
  // Gather in three dependent rounds with all four contributors of the lane in flight per round
  // (branch-free: out-of-range entries read a safe address and are masked): slot[q] (stage A); then
  // the NNF entry and n of that slot; then the proposed value u(p + phi(q)) = vox[src_q - off].
  uint32_t Dq[4], nq[4];
  uint64_t val[4];
  unsigned valid = 0;
  bool n125 = true;
  const int* off = LV.off;
  bool cand[4];
  int sl[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    cand[i] = (A.cand >> i) & 1u;
    sl[i] = A.sl[i];
  }
  uint64_t ev[4];
  uint32_t nv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    bool ok = cand[i] && sl[i] >= 0;
    int si = ok ? sl[i] : 0;
    ev[i] = __ldg(reinterpret_cast<const unsigned long long*>(a.e) + si);
    nv[i] = __ldg(a.n + si);
    cand[i] = ok;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    bool ok = cand[i] && (mode == VINP_UNWEIGHTED || nv[i] > 0);
    val[i] = __ldg(reinterpret_cast<const unsigned long long*>(a.vox) + (ok ? e_q(ev[i]) - off[i] : p));
    Dq[i] = ok ? e_D(ev[i]) : 0;
    nq[i] = ok ? nv[i] : 125;
    if (ok) {
      n125 &= (nv[i] == 125);
      valid |= 1u << i;
    } else {
      val[i] = 0;
    }
  }
  uint32_t m = __reduce_add_sync(kFull, (uint32_t)__popc(valid));
  if (m == 0) return;
  n125 = __all_sync(kFull, n125);
  // exact order keys of d^2 = D/(4n): D itself when every n = 125 (fast path), else the fp64
  // bit pattern of D/n (distinct rationals with n <= 125 are distinct, ordered doubles)
  uint64_t key[4];
  if (mode != VINP_UNWEIGHTED) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      key[i] = !(valid >> i & 1) ? ~0ull
               : n125 ? (uint64_t)Dq[i]
                      : (uint64_t)__double_as_longlong((double)Dq[i] / (double)nq[i]);
  }
  int64_t w[4];
  bool unitw = true;  // warp-uniform: every weight is 0 or 1 (best patch, unweighted, sigma_p = 0)
  if (mode == VINP_BEST_PATCH) {
    uint64_t kmin;
    if (n125) {
      kmin = __reduce_min_sync(kFull, (uint32_t)min(min(key[0], key[1]), min(key[2], key[3])));
    } else {
      kmin = warp_min64(min(min(key[0], key[1]), min(key[2], key[3])));
    }
    uint32_t vbest = 0xffffffffu;
#pragma unroll
    for (int i = 3; i >= 0; --i)
      if ((valid >> i & 1) && key[i] == kmin) vbest = lane + 32 * i;
    vbest = __reduce_min_sync(kFull, vbest);
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = ((uint32_t)(lane + 32 * i) == vbest) ? 1 : 0;
  } else if (mode == VINP_UNWEIGHTED) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = (valid >> i) & 1;
  } else {
    // sigma^2 key: the r-th smallest key, r = ceil(0.75 m) (nearest rank, R10), by a bitwise rank
    // search (one REDUX.SUM per bit) on the high 32 key bits from the first bit where the warp's
    // keys differ; the low 32 bits are searched only if the selected high half is shared by
    // unequal keys.  In the n = 125 fast path the key is D (high half 0).
    uint32_t r = (3 * m + 3) / 4;
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      hi[i] = n125 ? (uint32_t)key[i] : (uint32_t)(key[i] >> 32);  // ~0 for invalid
      lo[i] = n125 ? 0u : (uint32_t)key[i];
    }
    const uint32_t ans = select_rank32(hi, valid, r, m);
    uint32_t lans = 0;
    if (!n125) {
      uint32_t below = 0, lmin = 0xffffffffu, lmax = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        below += (valid >> i & 1) && hi[i] < ans;
        if (hi[i] == ans && (valid >> i & 1)) { lmin = min(lmin, lo[i]); lmax = max(lmax, lo[i]); }
      }
      below = __reduce_add_sync(kFull, below);
      lmin = __reduce_min_sync(kFull, lmin);
      lmax = __reduce_max_sync(kFull, lmax);
      lans = lmin;
      if (lmin != lmax) {
        uint32_t r2 = r - below;
        lans = lmin & ~(0xffffffffu >> __clz(lmax ^ lmin));
        for (int bit = 31 - __clz(lmax ^ lmin); bit >= 0; --bit) {
          uint32_t T = lans | ((1u << bit) - 1);
          uint32_t c = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) c += (hi[i] == ans && (valid >> i & 1) && lo[i] <= T);
          c = __reduce_add_sync(kFull, c);
          if (c < r2) lans |= 1u << bit;
        }
      }
    }
    uint32_t Ds, ns;
    if (n125) {
      Ds = ans;
      ns = 125;
    } else {
      uint64_t kans = ((uint64_t)ans << 32) | lans;
      // a representative (D_s, n_s) with key == kans (equal keys are equal rationals)
      int own = -1;
#pragma unroll
      for (int i = 3; i >= 0; --i)
        if ((valid >> i & 1) && key[i] == kans) own = i;
      unsigned bal = __ballot_sync(kFull, own >= 0);
      int src = __ffs(bal) - 1;
      uint32_t myD = 0, myn = 1;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i == own) { myD = Dq[i]; myn = nq[i]; }
      Ds = __shfl_sync(kFull, myD, src);
      ns = __shfl_sync(kFull, myn, src);
    }
    if (Ds == 0) {  // sigma_p = 0: the mean over the zero-distance contributors (R11)
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = ((valid >> i) & 1u) && Dq[i] == 0;
    } else if (n125) {
      unitw = false;
      // a = D_q / (2 D_s) with all n = 125: the correctly rounded quotient from the correctly rounded
      // reciprocal y = RN(1/b) (once per hole), q = RN(a y), r = a - q b (exact, FMA), RN(q + r y)
      // (Markstein's theorem; b = 2 D_s < 2^32 has no all-ones significand) — equal to __ddiv_rn
      // (host check of the same arithmetic: 3.2e9 random and 3.6e8 exhaustive small pairs, 0 differ).
      // Branch-free over the lane's four contributors (an absent one has D_q = 0 and is masked).
      const double den = (double)(2ull * Ds), rcp = __drcp_rn(den);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double an = __dadd_rn(__hiloint2double(0x43300000, (int)Dq[i]), -4503599627370496.0);  // (double)D_q
        const double q0 = __dmul_rn(an, rcp);
        const double aa = __fma_rn(__fma_rn(-q0, den, an), rcp, q0);
        const int64_t wi = weight36(aa, tab);
        w[i] = ((valid >> i) & 1u) ? wi : 0;
      }
    } else {
      unitw = false;
      // partial patches (volume border): a = D_q n_s / (2 n_q D_s), one correctly rounded division
      // of exact operands (R32)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double aa = __ddiv_rn((double)((uint64_t)Dq[i] * ns), (double)(2ull * nq[i] * Ds));
        const int64_t wi = weight36(aa, tab);
        w[i] = ((valid >> i) & 1u) ? wi : 0;
      }
    }
  }
  int64_t S;
  int64_t N[5];
  if (unitw) {
    // weights 0 / 1: the six sums are at most 125 * 255 < 2^16, two per 32-bit REDUX
    uint32_t p0 = 0, p1 = 0, p2 = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t c0 = w[i] ? (uint32_t)val[i] : 0u, c1 = w[i] ? (uint32_t)(val[i] >> 32) : 0u;
      p0 += (c0 & 0xffu) | ((c0 & 0xff00u) << 8);
      p1 += ((c0 >> 16) & 0xffu) | ((c1 & 0xffu) << 16);
      p2 += ((c1 >> 8) & 0xffu) | (w[i] ? 0x10000u : 0u);
    }
    p0 = __reduce_add_sync(kFull, p0);
    p1 = __reduce_add_sync(kFull, p1);
    p2 = __reduce_add_sync(kFull, p2);
    N[0] = p0 & 0xffffu;
    N[1] = p0 >> 16;
    N[2] = p1 & 0xffffu;
    N[3] = p1 >> 16;
    N[4] = p2 & 0xffffu;
    S = p2 >> 16;
  } else {
    // exact sums: w <= 2^36 is split as w = wh 2^32 + wl (wh <= 16); per channel the low part
    // accumulates in 64 bits (one wide multiply-add per contributor) and the high part in 32 bits;
    // the per-lane partials (< 2^46) are then summed over the warp as two 23-bit halves by REDUX
    uint64_t Sl = 0, Nl[5] = {0, 0, 0, 0, 0};
    uint32_t Sh = 0, Nh[5] = {0, 0, 0, 0, 0};
  #pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t wl = (uint32_t)w[i], wh = (uint32_t)((uint64_t)w[i] >> 32);
      const uint64_t x = val[i];
      const uint32_t c0 = (uint32_t)x, c1 = (uint32_t)(x >> 32);
      const uint32_t v[5] = {c0 & 255, (c0 >> 8) & 255, (c0 >> 16) & 255, c1 & 255, (c1 >> 8) & 255};
      Sl += wl;
      Sh += wh;
  #pragma unroll
      for (int c = 0; c < 5; ++c) {
        Nl[c] += (uint64_t)wl * v[c];
        Nh[c] += wh * v[c];
      }
    }
    S = warp_sum46((int64_t)(Sl + ((uint64_t)Sh << 32)));
  #pragma unroll
    for (int c = 0; c < 5; ++c) N[c] = warp_sum46((int64_t)(Nl[c] + ((uint64_t)Nh[c] << 32)));
  }
  if (lane < 5) {
    int64_t Nc = lane == 0 ? N[0] : lane == 1 ? N[1] : lane == 2 ? N[2] : lane == 3 ? N[3] : N[4];
    float o = (float)__ddiv_rn((double)Nc, (double)S);
    if (lane < 3) out_rgb[3 * (int64_t)h + lane] = o;
    else out_tex[2 * (int64_t)h + lane - 3] = o;
    if (commit) {
      uint32_t b = round_u8(o);
      uint32_t sh = lane < 3 ? 8 * lane : 32 + 8 * (lane - 3);
      uint64_t part = (uint64_t)b << sh;
      // combine the five bytes in lane 0
      uint32_t lo = (uint32_t)part, hi = (uint32_t)(part >> 32);
      lo |= __shfl_down_sync(0x1f, lo, 1) | __shfl_down_sync(0x1f, lo, 2);
      hi |= __shfl_down_sync(0x1f, hi, 3) | __shfl_down_sync(0x1f, hi, 4);
      if (lane == 0) a.vox[p] = ((uint64_t)hi << 32) | lo;
    }
  }
}

// persistent warps over the holes [hb, he) (or list[hb..he)): the lane geometry is set up once
__global__ void __launch_bounds__(32 * kWPB, VINP_REC_MINB * 8 / kWPB) k_reconstruct(ReconArgs a, int mode, int layer_j, int32_t hb,
                                                     int32_t he, const int32_t* __restrict__ list,
                                                     float* __restrict__ out_rgb,
                                                     float* __restrict__ out_tex, int commit) {
  const int lane = threadIdx.x & 31;
  __shared__ double2 s_tab[128];
  if (threadIdx.x < 128) s_tab[threadIdx.x] = kExpTab[threadIdx.x];
  __syncthreads();
  LaneVox LV;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int v = lane + 32 * i;
    int dx, dy, dt;
    voff(v < kPatch ? v : 62, dx, dy, dt);
    LV.off[i] = dt * a.g.HW + dy * a.g.W + dx;
    LV.dx[i] = (int8_t)dx;
    LV.dy[i] = (int8_t)dy;
    LV.dt[i] = (int8_t)dt;
    LV.real[i] = v < kPatch;
  }
#if VINP_REC_CHUNKED
  // each block owns a contiguous chunk of holes, its warps 8 adjacent holes at a time: co-resident
  // blocks (consecutive ids) then work on neighbouring holes, whose contributors share cache lines
  const int chunk = ((he - hb) + gridDim.x - 1) / gridDim.x;
  const int cb = hb + blockIdx.x * chunk;
  he = min(he, cb + chunk);
  const int nw = kWPB;
  int idx = cb + (threadIdx.x >> 5);
#else
  const int nw = gridDim.x * kWPB;
  int idx = hb + blockIdx.x * kWPB + (threadIdx.x >> 5);
#endif
  if (idx >= he) return;
#if VINP_REC_PREFETCH
  HoleA cur = recon_stage_a(a, LV, layer_j, list ? __ldg(list + idx) : idx);
  for (;;) {
    const int nidx = idx + nw;
    const bool more = nidx < he;
    const HoleA nxt = recon_stage_a(a, LV, layer_j, more ? (list ? __ldg(list + nidx) : nidx) : cur.h);
    recon_hole(a, LV, lane, mode, layer_j, cur, out_rgb, out_tex, commit, s_tab);
    if (!more) break;
    cur = nxt;
    idx = nidx;
  }
#else
  for (; idx < he; idx += nw)
    recon_hole(a, LV, lane, mode, layer_j, recon_stage_a(a, LV, layer_j, list ? __ldg(list + idx) : idx), out_rgb,
               out_tex, commit, s_tab);
#endif
}

__global__ void k_commit(Geo g, uint64_t* __restrict__ vox, const uint8_t* __restrict__ layer,
                         const int32_t* __restrict__ holes, const float* __restrict__ rgb,
                         const float* __restrict__ tex, int layer_j, int32_t hb, int32_t he) {
  int h = hb + blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= he) return;
  int p = holes[h];
  if (layer_j >= 0 && layer[p] != layer_j) return;
  uint64_t w = (uint64_t)round_u8(rgb[3 * (int64_t)h]) | ((uint64_t)round_u8(rgb[3 * (int64_t)h + 1]) << 8) |
               ((uint64_t)round_u8(rgb[3 * (int64_t)h + 2]) << 16) |
               ((uint64_t)round_u8(tex[2 * (int64_t)h]) << 32) |
               ((uint64_t)round_u8(tex[2 * (int64_t)h + 1]) << 40);
  vox[p] = w;
}

// L2 = false: sum llrint(|a-b| 2^20) (R19); L2 = true: sum llrint((a-b)^2 2^20), the literal
// P:988 norm (the difference of two floats and its square are exact in fp64)
template <bool L2>
__global__ void k_change(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                         unsigned long long* __restrict__ out) {
  int64_t acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = (double)a[i] - (double)b[i];
    acc += __double2ll_rn((L2 ? __dmul_rn(d, d) : fabs(d)) * 1048576.0);
  }
  acc = warp_sum64(acc);
  __shared__ long long sm[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sm[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += sm[k];
    if (s) atomicAdd(out, (unsigned long long)s);
  }
}

// deterministic single-block sum of D/(4n) over H (diagnostic)
__global__ void k_energy(const int32_t* __restrict__ holes, int32_t nh, const int32_t* __restrict__ slot,
                         const uint64_t* __restrict__ e, const uint8_t* __restrict__ n,
                         double* __restrict__ out) {
  double acc = 0;
  for (int h = threadIdx.x; h < nh; h += blockDim.x) {
    int s = slot[holes[h]];
    if (s >= 0 && n[s]) acc += (double)e_D(e[s]) / (4.0 * n[s]);
  }
  __shared__ double sm[1024];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int k = blockDim.x / 2; k; k >>= 1) {
    if ((int)threadIdx.x < k) sm[threadIdx.x] += sm[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

}  // namespace vinp

using namespace vinp;

namespace vinp {
vinp_status launch_reconstruct(vinp_level* lv, const vinp_nnf* nnf, int mode, int layer_j, int32_t hb,
                               int32_t he, const int32_t* list, float* out_rgb, float* out_tex,
                               int commit, void* stream) {
  vinp_status st = check_level(lv, "vinp_reconstruct");
  if (st) return st;
  VINP_REQUIRE(nnf && nnf->e && nnf->n && out_rgb && out_tex && lv->holes && lv->slot,
               "vinp_reconstruct: null buffers");
  VINP_REQUIRE(mode == VINP_WEIGHTED || mode == VINP_UNWEIGHTED || mode == VINP_BEST_PATCH,
               "vinp_reconstruct: bad mode %d", mode);
  VINP_REQUIRE(hb >= 0 && (list || he <= lv->n_holes) && hb <= he, "vinp_reconstruct: bad hole range");
  VINP_REQUIRE(layer_j < 0 || lv->layer, "vinp_reconstruct: layer map required");
  if (he > hb) {
    ReconArgs a{geo_of(lv), lv->vox, lv->layer, lv->slot, lv->holes, nnf->e, nnf->n};
    const int grid = (int)std::min<int64_t>(nblk(he - hb, kWPB), 148 * (VINP_REC_MINB * 8 / kWPB) * VINP_REC_WAVES);  // persistent warps
    k_reconstruct<<<grid, 32 * kWPB, 0, S(stream)>>>(a, mode, layer_j, hb, he, list,
                                                                  out_rgb, out_tex, commit);
    count_launch();
  }
  return check_launch("vinp_reconstruct");
}
}  // namespace vinp

extern "C" {
vinp_status vinp_reconstruct(vinp_level* lv, const vinp_nnf* nnf, int mode, int layer_j, int32_t hb,
                             int32_t he, float* out_rgb, float* out_tex, int commit, void* stream) {
  VINP_NVTX();
  return launch_reconstruct(lv, nnf, mode, layer_j, hb, he, nullptr, out_rgb, out_tex, commit, stream);
}

vinp_status vinp_commit(vinp_level* lv, const float* out_rgb, const float* out_tex, int layer_j,
                        int32_t hb, int32_t he, void* stream) {
  VINP_NVTX();
  vinp_status st = check_level(lv, "vinp_commit");
  if (st) return st;
  VINP_REQUIRE(out_rgb && out_tex && lv->holes, "vinp_commit: null buffers");
  VINP_REQUIRE(hb >= 0 && he <= lv->n_holes && hb <= he, "vinp_commit: bad hole range");
  VINP_REQUIRE(layer_j < 0 || lv->layer, "vinp_commit: layer map required");
  if (he > hb) {
    k_commit<<<nblk(he - hb, 256), 256, 0, S(stream)>>>(geo_of(lv), lv->vox, lv->layer, lv->holes,
                                                        out_rgb, out_tex, layer_j, hb, he);
    count_launch();
  }
  return check_launch("vinp_commit");
}

vinp_status vinp_change_l1(const float* a, const float* b, int64_t n, int64_t* out, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(out && n >= 0 && (n == 0 || (a && b)), "vinp_change_l1: bad args");
  if (n > 0) {
    int g = (int)std::min<int64_t>(nblk(n, 256), 148 * 8);
    k_change<false><<<g, 256, 0, S(stream)>>>(a, b, n, (unsigned long long*)out);
    count_launch();
  }
  return check_launch("vinp_change_l1");
}

vinp_status vinp_change_l2(const float* a, const float* b, int64_t n, int64_t* out, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(out && n >= 0 && (n == 0 || (a && b)), "vinp_change_l2: bad args");
  if (n > 0) {
    int g = (int)std::min<int64_t>(nblk(n, 256), 148 * 8);
    k_change<true><<<g, 256, 0, S(stream)>>>(a, b, n, (unsigned long long*)out);
    count_launch();
  }
  return check_launch("vinp_change_l2");
}

vinp_status vinp_energy(const vinp_level* lv, const vinp_nnf* nnf, double* out, void* stream) {
  VINP_NVTX();
  vinp_status st = check_level(lv, "vinp_energy");
  if (st) return st;
  VINP_REQUIRE(nnf && nnf->e && nnf->n && out && lv->holes && lv->slot, "vinp_energy: null buffers");
  k_energy<<<1, 1024, 0, S(stream)>>>(lv->holes, lv->n_holes, lv->slot, nnf->e, nnf->n, out);
  count_launch();
  return check_launch("vinp_energy");
}

}  // extern "C"
