// common.cuh — shared device helpers of libvinp (sm_100a).  Not shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include <nvtx3/nvToolsExt.h>

#include "vinp.h"

namespace vinp {

// One NVTX range per C-ABI call (header-only NVTX v3: without an attached tool the push / pop are
// a null-pointer test each), so nsys / ncu --nvtx can attribute kernels to the call that launched
// them.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define VINP_NVTX() ::vinp::NvtxRange vinp_nvtx_range_(__func__)

constexpr int kPatch = 125;   // 5x5x5
constexpr int kR = 2;         // patch radius
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- host-side error plumbing
void set_error(const char* fmt, ...);
vinp_status check_launch(const char* what);
void count_launch(int n = 1);

#define VINP_REQUIRE(cond, ...)          \
  do {                                   \
    if (!(cond)) {                       \
      ::vinp::set_error(__VA_ARGS__);    \
      return VINP_E_INVALID;             \
    }                                    \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline vinp_status check_level(const vinp_level* lv, const char* who) {
  if (!lv || !lv->vox || !lv->flags) {
    set_error("%s: null level or buffers", who);
    return VINP_E_INVALID;
  }
  if (lv->W < 1 || lv->H < 1 || lv->T < 1 || (int64_t)lv->W * lv->H * lv->T >= (1ll << 31)) {
    set_error("%s: bad dims %dx%dx%d", who, lv->W, lv->H, lv->T);
    return VINP_E_UNSUPPORTED;
  }
  return VINP_OK;
}

// internal launchers with an optional index list (list[i] = slot / hole index, i in [b, e))
vinp_status launch_evaluate(const vinp_level* lv, vinp_nnf* nnf, const vinp_params* prm, int kb,
                            int only_layer, int32_t b, int32_t e, const int32_t* list,
                            unsigned long long* counter, void* stream);
vinp_status launch_propagate(const vinp_level* lv, const vinp_nnf* in, vinp_nnf* out,
                             const vinp_params* prm, int step, int sign, int kb, int only_layer,
                             int32_t b, int32_t e, int pass, int since, const int32_t* list,
                             unsigned long long* counter, void* stream);
vinp_status launch_random_search(const vinp_level* lv, const vinp_nnf* in, vinp_nnf* out,
                                 const vinp_params* prm, uint32_t outer_code, int pm_iter, int kb,
                                 int only_layer, int32_t b, int32_t e, int pass, const int32_t* list,
                                 unsigned long long* counter, void* stream);

// Pass numbering of one ANN search for the R41 stale skip (host side): evaluate = pass 0, then
// 1, 2, ... in schedule order; since(step, sign) = the index of the last earlier propagation pass
// with that (step, sign), 0 if none.
struct PassClock {
  int pass = 1;
  int n = 0;
  int key_step[64], key_sign[64], last[64];
  int since(int step, int sign) const {
    for (int i = 0; i < n; ++i)
      if (key_step[i] == step && key_sign[i] == sign) return last[i];
    return 0;
  }
  void tick(int step, int sign) {  // sign 2 = a random-search pass
    if (sign != 2) {
      int i = 0;
      while (i < n && !(key_step[i] == step && key_sign[i] == sign)) ++i;
      if (i == n && n < 64) {
        key_step[n] = step;
        key_sign[n] = sign;
        ++n;
      }
      if (i < 64) last[i] = pass;
    }
    ++pass;
  }
};
vinp_status launch_reconstruct(vinp_level* lv, const vinp_nnf* nnf, int mode, int layer_j, int32_t hb,
                               int32_t he, const int32_t* list, float* out_rgb, float* out_tex,
                               int commit, void* stream);

// ---------------------------------------------------------------- geometry
// Division by the invariant W and HW via multiply-high: for 0 <= n < 2^31 and d >= 1,
// floor(n / d) = (n * m) >> (32 + s) with s = ceil(log2 d), m = floor(2^(32+s) / d) + 1
// (error n*(m - 2^(32+s)/d)/2^(32+s) < 2^-(1+s) <= 1/(2d), below the gap to the next integer).
struct Geo {
  int W, H, T;
  int HW;
  uint64_t mW, mHW;
  int sW, sHW;
};
inline void magic_of(uint32_t d, uint64_t& m, int& s) {
  s = 0;
  while ((1ull << s) < d) ++s;
  m = ((1ull << (32 + s)) / d) + 1;
}
inline Geo geo_of(const vinp_level* lv) {
  Geo g{lv->W, lv->H, lv->T, lv->W * lv->H, 0, 0, 0, 0};
  magic_of((uint32_t)g.W, g.mW, g.sW);
  magic_of((uint32_t)g.HW, g.mHW, g.sHW);
  return g;
}
__device__ __forceinline__ int fdiv(uint32_t n, uint64_t m, int s) {
  return (int)(((uint64_t)n * m) >> (32 + s));  // n < 2^31, m <= 2^33: the product fits in 64 bits
}

__device__ __forceinline__ void decode(const Geo& g, int p, int& x, int& y, int& t) {
  t = fdiv((uint32_t)p, g.mHW, g.sHW);
  int r = p - t * g.HW;
  y = fdiv((uint32_t)r, g.mW, g.sW);
  x = r - y * g.W;
}

__device__ __forceinline__ bool inside(const Geo& g, int x, int y, int t) {
  return (unsigned)x < (unsigned)g.W && (unsigned)y < (unsigned)g.H && (unsigned)t < (unsigned)g.T;
}

// patch offset index v in [0,125): dx = v%5-2, dy = (v/5)%5-2, dt = v/25-2 (t-major order)
__device__ __forceinline__ void voff(int v, int& dx, int& dy, int& dt) {
  dt = v / 25 - 2;
  int r = v % 25;
  dy = r / 5 - 2;
  dx = r % 5 - 2;
}

// ---------------------------------------------------------------- Philox4x32-10
__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}
enum { kStreamInit = 1, kStreamRS = 2, kStreamRepair = 3 };
__device__ __forceinline__ uint4 draw(uint32_t p, uint32_t k, int level, int stream, int i,
                                      uint32_t oc, uint64_t seed) {
  return philox(make_uint4(p, k, ((uint32_t)level << 24) | ((uint32_t)stream << 16) | (uint32_t)i, oc),
                (uint32_t)seed, (uint32_t)(seed >> 32));
}

// ---------------------------------------------------------------- NNF mirrors (NEXT #4 stage 2)
// Passed by value to the pass kernels: the epilogue stores every written entry into the peer
// copies too (P2P stores), and e through the NVLS multicast address when there is one.
struct Mirror {
  int n;
  uint64_t* e[VINP_MAX_PEERS];
  uint8_t* nn[VINP_MAX_PEERS];
  uint8_t* st[VINP_MAX_PEERS];
  uint64_t* mc_e;
};
inline Mirror mirror_of(const vinp_nnf* f) {
  Mirror m{};
  if (f && f->mirror) {
    const vinp_mirror* s = f->mirror;
    m.n = s->n_peers;
    for (int i = 0; i < s->n_peers && i < VINP_MAX_PEERS; ++i) {
      m.e[i] = s->e[i];
      m.nn[i] = s->n[i];
      m.st[i] = s->stamp[i];
    }
    m.mc_e = s->mc_e;
  }
  return m;
}
__device__ __forceinline__ void multimem_st_u64(uint64_t* mc, uint64_t v) {
  asm volatile("multimem.st.relaxed.sys.global.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
__device__ __forceinline__ void put_e(uint64_t* __restrict__ dst, const Mirror& m, int s, uint64_t v) {
  dst[s] = v;
  if (m.mc_e) {
    multimem_st_u64(m.mc_e + s, v);
  } else {
    for (int i = 0; i < m.n; ++i) m.e[i][s] = v;
  }
}
__device__ __forceinline__ void put_u8(uint8_t* __restrict__ dst, uint8_t* const* peers, int np, int s,
                                       uint8_t v) {
  dst[s] = v;
  for (int i = 0; i < np; ++i)
    if (peers[i]) peers[i][s] = v;
}

// ---------------------------------------------------------------- NNF entry packing
__device__ __forceinline__ uint64_t pack_e(uint32_t D, int32_t q) {
  return ((uint64_t)D << 32) | (uint32_t)q;
}
__device__ __forceinline__ uint32_t e_D(uint64_t e) { return (uint32_t)(e >> 32); }
__device__ __forceinline__ int32_t e_q(uint64_t e) { return (int32_t)(uint32_t)e; }

// ---------------------------------------------------------------- warp-per-target patch state
// Lane l owns patch voxels v = l + 32 i, i = 0..3 (v < 125).  off[i] is the linear offset of v,
// identical for the target patch around p and the source patch around q (same geometry).
struct PatchLanes {
  int off[4];
  int dx[4], dy[4], dt[4];
  bool live[4];  // v < 125
};
__device__ __forceinline__ void init_lanes(PatchLanes& L, const Geo& g, int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int v = lane + 32 * i;
    L.live[i] = v < kPatch;
    int dx, dy, dt;
    voff(L.live[i] ? v : 62, dx, dy, dt);
    L.dx[i] = dx; L.dy[i] = dy; L.dt[i] = dt;
    L.off[i] = dt * g.HW + dy * g.W + dx;
  }
}

struct TargetPatch {
  uint32_t c[4], t[4];  // colour / texture words of the target voxels
  unsigned mask;        // bit i: voxel i in Omega and in K
};

// K = Omega (kb < 0) or {r : layer(r) < kb}
__device__ __forceinline__ void load_target(TargetPatch& tp, const PatchLanes& L, const Geo& g,
                                            const uint64_t* __restrict__ vox,
                                            const uint8_t* __restrict__ layer, int kb, int p,
                                            int px, int py, int pt) {
  tp.mask = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    tp.c[i] = 0; tp.t[i] = 0;
    if (L.live[i] && inside(g, px + L.dx[i], py + L.dy[i], pt + L.dt[i])) {
      int r = p + L.off[i];
      bool known = kb < 0 || layer[r] < kb;
      if (known) {
        uint64_t w = __ldg(reinterpret_cast<const unsigned long long*>(vox) + r);
        tp.c[i] = (uint32_t)w;
        tp.t[i] = (uint32_t)(w >> 32);
        tp.mask |= 1u << i;
      }
    }
  }
}

__device__ __forceinline__ uint32_t voxel_cost(uint32_t tc, uint32_t tt, uint64_t s, int lambda) {
  uint32_t dc = __vabsdiffu4(tc, (uint32_t)s);
  uint32_t dtx = __vabsdiffu4(tt, (uint32_t)(s >> 32));
  uint32_t cc = __dp4a(dc, dc, 0u);
  uint32_t tc2 = __dp4a(dtx, dtx, 0u);
  return 4u * cc + (uint32_t)lambda * tc2;
}

// D(p, q) for the whole warp (all lanes return the same value).  q must be in D~.
__device__ __forceinline__ uint32_t warp_ssd(const TargetPatch& tp, const PatchLanes& L,
                                             const uint64_t* __restrict__ vox, int q, int lambda) {
  uint32_t acc = 0;
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(vox);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (tp.mask & (1u << i)) {
      uint64_t s = __ldg(v + q + L.off[i]);
      acc += voxel_cost(tp.c[i], tp.t[i], s, lambda);
    }
  }
  return __reduce_add_sync(kFull, acc);
}


__device__ __forceinline__ bool is_source(const Geo& g, const uint8_t* __restrict__ flags, int x,
                                          int y, int t) {
  if (!inside(g, x, y, t)) return false;
  return (__ldg(flags + (t * g.HW + y * g.W + x)) & 2) != 0;
}

}  // namespace vinp
