// ann.cu — PatchMatch ANN search on sm_100a: NNF init / upsample / evaluate (a5), Jacobi jump
// propagation (a6), Philox random search (a7), the Alg. 1 schedule (a8), exact brute force (a13,
// CUDA-core form), and the SSD / Philox test hooks.
//
// Execution model: evaluate and propagation run thread-per-target (lane = an
// x-adjacent target, so the coherent candidate gathers coalesce), random search runs 5-lane column
// groups over a per-warp pair queue (incoherent candidates), onion-layer propagation runs warp per
// target (short latency chain for small launches).  Distances are exact integers (VABSDIFF4 +
// IDP.4A per colour / texture word); early aborts change no comparison, and neither do the three
// exact savings: stale propagation candidates (R41), R41-active passes over the targets that read
// a changed entry only (R41b: k_prop_mark, k_prop_compact), and the patch-sum lower bound that
// rejects candidates before any patch row is read (R42: k_patch_sums_*).  Every pass reads NNF
// buffer `in` and writes `out` (double buffering): no atomics on the NNF, results independent of
// scheduling.
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace vinp {

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }
constexpr int kWarpsPerBlock = 8;

struct LevelArgs {
  Geo g;
  const uint64_t* vox;
  const uint8_t* flags;
  const uint8_t* layer;
  const int32_t* slot;
  const int32_t* targets;
  const int32_t* sources;
  int32_t n_sources;
  int level;
  const uint4* psum;  // R42 patch sums, or null
  int32_t n_targets;
};
static LevelArgs args_of(const vinp_level* lv) {
  return LevelArgs{geo_of(lv), lv->vox,     lv->flags,     lv->layer, lv->slot,
                   lv->targets, lv->sources, lv->n_sources, lv->level,
                   reinterpret_cast<const uint4*>(lv->psum), lv->n_targets};
}

__device__ __forceinline__ int lin(const Geo& g, int x, int y, int t) {
  return t * g.HW + y * g.W + x;
}

__device__ __forceinline__ void flush_count(unsigned long long* counter, unsigned cnt) {
  if (counter && cnt) atomicAdd(counter, (unsigned long long)cnt);
}

// ------------------------------------------------------------------ a5: random init
__global__ void k_init_random(LevelArgs a, uint64_t* __restrict__ e_out, uint8_t* __restrict__ n_out,
                              uint64_t seed, uint32_t oc, int32_t b, int32_t e) {
  int s = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= e) return;
  int p = a.targets[s];
  uint4 u = draw((uint32_t)p, 0, a.level, kStreamInit, 0, oc, seed);
  int q = a.sources[__umulhi(u.x, (uint32_t)a.n_sources)];
  e_out[s] = pack_e(0, q);
  n_out[s] = 0;
}

// ------------------------------------------------------------------ a5: upsample (+ R21 repair)
__global__ void k_upsample(LevelArgs c, const uint64_t* __restrict__ ce, LevelArgs f,
                           uint64_t* __restrict__ fe, uint8_t* __restrict__ fn, uint64_t seed,
                           int32_t b, int32_t e) {
  int s = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= e) return;
  int p = f.targets[s];
  int px, py, pt;
  decode(f.g, p, px, py, pt);
  int cx = px >> 1, cy = py >> 1;
  int cs = c.slot[lin(c.g, cx, cy, pt)];
  int q = -1;
  if (cs >= 0) {
    int cq = e_q(ce[cs]);
    int qx, qy, qt;
    decode(c.g, cq, qx, qy, qt);
    int fx = px + 2 * (qx - cx), fy = py + 2 * (qy - cy), ft = pt + (qt - pt);
    if (is_source(f.g, f.flags, fx, fy, ft)) q = lin(f.g, fx, fy, ft);
  }
  if (q < 0) {
    uint4 u = draw((uint32_t)p, 0, f.level, kStreamRepair, 0, 0, seed);
    q = f.sources[__umulhi(u.x, (uint32_t)f.n_sources)];
  }
  fe[s] = pack_e(0, q);
  fn[s] = 0;
}

#ifndef VINP_EVAL_BLOCK
#define VINP_EVAL_BLOCK 64  // shorter tails (measured: level-1 evaluate 13.5 -> 12.3 ms per step vs 256)
#endif
#ifndef VINP_RS_WPB
#define VINP_RS_WPB 2  // warps per block for <= 12 candidates (measured: 8 -> 2 saves 3% per step)
#endif
#ifndef VINP_PROP_BLOCK
#define VINP_PROP_BLOCK 128  // smaller blocks shorten the tail of every pass (measured: -2% per step vs 256)
#endif
#ifndef VINP_PROP_BLOCK_MID
#define VINP_PROP_BLOCK_MID 64  // launches below VINP_PROP_BIG targets (levels >= 2 of c5): -3 ms per step
#endif
#ifndef VINP_PROP_BIG
#define VINP_PROP_BIG (1 << 23)
#endif
#ifndef VINP_MINB
#define VINP_MINB 4
#endif
#ifndef VINP_PROP_MINB
#define VINP_PROP_MINB 4
#endif
#ifndef VINP_PROP_FRAME_MAJOR
#define VINP_PROP_FRAME_MAJOR 1
#endif
#ifndef VINP_PROP_SPARSE
#define VINP_PROP_SPARSE 48  // warps with at most this many live propagation candidates: group path (A/B: 12 -> 48 = -4% per ANN search)
#endif
#ifndef VINP_PROP_LIGHT
#define VINP_PROP_LIGHT 1  // R41-active propagation passes run the light kernel
#endif
#ifndef VINP_PROP_LIGHT_MINB
#define VINP_PROP_LIGHT_MINB 8  // 128-thread blocks per SM the light kernel is compiled for (A/B: 8 < 12, 16)
#endif
#ifndef VINP_RS_ORDER
#define VINP_RS_ORDER 1  // random-search pair list: 0 lane-major, 1/2 rank-major (ascending/descending); A/B: 1 is -0.7%
#endif
#ifndef VINP_RS_GEN_CHUNK
#define VINP_RS_GEN_CHUNK 4  // random-search candidate generation: D~ flag loads in flight together per chunk
#endif
#ifndef VINP_ACTIVE_MIN
#define VINP_ACTIVE_MIN (1 << 20)
#endif
#ifndef VINP_PROP_LB
#define VINP_PROP_LB 1  // R42 lower bound in propagation too
#endif
#ifndef VINP_RS_SMALL
#define VINP_RS_SMALL (148 * 32 * 8)  // random-search launches below this many targets: 8 per warp
#endif

// ------------------------------------------------------------------ pair evaluation by column groups
// Random search and sparse propagation warps, evaluation by 5-lane column groups: lanes 5g..5g+4 (g < 6) evaluate one
// (target, candidate) pair, lane k owning patch column dx = k - 2, so every row of a patch is one
// 40-byte gather per group.  Pairs come from the warp's flattened candidate list (owner lane =
// target, rank order); each group takes the next unassigned pair as soon as its own aborts or
// completes.  Exact partial-distance elimination after every frame dt (25 voxels): the group sum
// is all-reduced over its 5 lanes (3 shuffles) and checked against the owner's current minimum.
__device__ __forceinline__ uint32_t sum5(uint32_t x, int base, int k) {
  uint32_t s1 = x + __shfl_sync(kFull, x, base + (k + 1) % 5);
  uint32_t s2 = s1 + __shfl_sync(kFull, s1, base + (k + 2) % 5);
  return s2 + __shfl_sync(kFull, x, base + (k + 4) % 5);
}

// Evaluation of a warp's (candidate q, owner lane) pair list by 5-lane column groups: lanes
// 5g..5g+4 (g < 6) evaluate one pair, lane k owning patch column dx = k - 2, so every row of a
// patch is one 40-byte gather per group.  The owner lane holds its target (p, px, py, pt) and its
// running best (bestD, bestq), initially the incumbent; pairs of one owner are in rank order.
// Out-of-volume voxels of a border target contribute nothing (K = Omega).
__device__ __forceinline__ void group_eval(const LevelArgs& a, const int2* pairs, const int P,
                                           const int lane, const int p, const int px, const int py,
                                           const int pt, const int lambda, uint32_t& bestD,
                                           int& bestq) {
  const int g = lane / 5, k = lane - 5 * (lane / 5), gbase = 5 * g, dx = k - 2;
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox);
  // Each 5-lane group g < 6 walks the warp's pair list on its own: one frame of its current pair
  // per loop iteration, and as soon as the pair aborts or completes the group takes the next
  // unassigned pair, so a surviving pair never holds other groups idle.  Sequential application
  // in rank order with strict improvement (R25) equals the lexicographic minimum of (D, pair index)
  // over {incumbent (D_inc, -1)} + candidates, the index being the candidate's rank among its
  // owner's candidates (carried in the pair: y = rank << 5 | owner lane), so the list may be in any
  // order; a pair is dropped once its partial sum proves it cannot reach that minimum (partial >
  // best D, or == best D with a later rank): exact (R35).
  int bestJ = -1;
  int j = -1, dtc = -2, t = 0, pi = 0, ty = 0, tt = 0, sq = 0;
  bool colok = false;
  uint32_t accc = 0, acct = 0;
  int next = 0;
  const int gsrc = gbase < 30 ? gbase : 0;
  for (;;) {
    // hand out pairs to the groups that need one (in group order)
    bool need = g < 6 && j < 0 && next < P;
    unsigned nb = __ballot_sync(kFull, need && k == 0);
    if (nb) {
      int jj = next + __popc(nb & ((1u << gbase) - 1u));
      bool take = need && jj < P;
      int2 pr = take ? pairs[jj] : make_int2(0, lane);
      int src = take ? (pr.y & 31) : lane;
      int npi = __shfl_sync(kFull, p, src), ntx = __shfl_sync(kFull, px, src);
      int nty = __shfl_sync(kFull, py, src), ntt = __shfl_sync(kFull, pt, src);
      if (take) {
        j = pr.y >> 5;  // the candidate's rank among its owner's candidates (R25 tie key)
        t = pr.y & 31;
        sq = pr.x;
        pi = npi;
        ty = nty;
        tt = ntt;
        colok = (unsigned)(ntx + dx) < (unsigned)a.g.W;
        dtc = -2;
        accc = acct = 0;
      }
      next = min(P, next + __popc(nb));
    }
    bool active = j >= 0;
    if (!__any_sync(kFull, active)) break;
    // one frame of the current pair: all 10 gathers first, then the arithmetic
    bool tok = active && colok && (unsigned)(tt + dtc) < (unsigned)a.g.T;
    int ro[5];
    bool okr[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      ro[r] = dtc * a.g.HW + (r - 2) * a.g.W + dx;
      okr[r] = tok && (unsigned)(ty + r - 2) < (unsigned)a.g.H;
    }
    uint64_t tv[5], sv[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      tv[r] = __ldg(v + pi + (okr[r] ? ro[r] : 0));
      sv[r] = __ldg(v + sq + (okr[r] ? ro[r] : 0));
    }
    uint32_t tD = __shfl_sync(kFull, bestD, active ? t : lane);
    int tJ = __shfl_sync(kFull, bestJ, active ? t : lane);
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      uint64_t tw = okr[r] ? tv[r] : 0ull, sw = okr[r] ? sv[r] : 0ull;
      uint32_t dc = __vabsdiffu4((uint32_t)tw, (uint32_t)sw);
      uint32_t dtx = __vabsdiffu4((uint32_t)(tw >> 32), (uint32_t)(sw >> 32));
      accc = __dp4a(dc, dc, accc);
      acct = __dp4a(dtx, dtx, acct);
    }
    uint32_t tot = sum5(4u * accc + (uint32_t)lambda * acct, gsrc, k);
    bool dead = active && (tot > tD || (tot == tD && j > tJ));
    bool win = active && !dead && dtc == 2;
    unsigned wb = __ballot_sync(kFull, win && k == 0);
    while (wb) {  // apply this iteration's completed pairs (several may share an owner)
      int src = __ffs(wb) - 1;
      wb &= wb - 1u;
      uint32_t D = __shfl_sync(kFull, tot, src);
      int jw = __shfl_sync(kFull, j, src);
      int qw = __shfl_sync(kFull, sq, src);
      int own = __shfl_sync(kFull, t, src);
      if (lane == own && (D < bestD || (D == bestD && jw < bestJ))) {
        bestD = D;
        bestJ = jw;
        bestq = qw;
      }
    }
    if (active) {
      if (dead || dtc == 2)
        j = -1;
      else
        ++dtc;
    }
  }
}

// ------------------------------------------------------------------ thread-per-target SSD
// Used where candidates are spatially coherent (evaluate, propagation): lane l of a warp owns
// target slot s0 + l, and consecutive slots are x-adjacent voxels, whose candidate sources are
// usually x-adjacent too.  Each of the 125 gathers of a patch is then one coalesced warp load of
// ~32 adjacent 8-byte voxels (2-3 L1 lines), addressed as row pointer + immediate offset.
// Exact partial-distance elimination after every frame of 25 voxels (SPEC: early abort that
// changes no comparison): a lane drops its candidate once the partial sum reaches `thr`.
// `full` = 1: every voxel of N_p is in Omega and K (interior target, K = Omega).
#define VINP_ACC(T, S)                                                        \
  {                                                                           \
    uint32_t dc = __vabsdiffu4((uint32_t)(T), (uint32_t)(S));                 \
    uint32_t dx_ = __vabsdiffu4((uint32_t)((T) >> 32), (uint32_t)((S) >> 32)); \
    accc = __dp4a(dc, dc, accc);                                              \
    acct = __dp4a(dx_, dx_, acct);                                            \
  }
// R42 helpers: channel sums of a voxel word, packed patch sums, full-patch test
__device__ __forceinline__ void vox_add(uint64_t w, uint32_t (&s)[5]) {
  const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
  s[0] = __dp4a(lo, 0x00000001u, s[0]);
  s[1] = __dp4a(lo, 0x00000100u, s[1]);
  s[2] = __dp4a(lo, 0x00010000u, s[2]);
  s[3] = __dp4a(hi, 0x00000001u, s[3]);
  s[4] = __dp4a(hi, 0x00000100u, s[4]);
}
__device__ __forceinline__ uint4 psum_pack(const uint32_t (&s)[5]) {
  return make_uint4(s[0] | (s[1] << 16), s[2] | (s[3] << 16), s[4], 0u);
}
__device__ __forceinline__ bool interior(const Geo& g, int x, int y, int t) {
  return x >= 2 && x < g.W - 2 && y >= 2 && y < g.H - 2 && t >= 2 && t < g.T - 2;
}

template <bool ABORT, bool SUMS = false>
__device__ __forceinline__ uint32_t thread_ssd(const LevelArgs& a, int p, int px, int py, int pt,
                                               int q, int lambda, int kb, bool full, uint32_t thr,
                                               bool& alive, uint32_t* psums = nullptr) {
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox);
  uint32_t accc = 0, acct = 0;
#pragma unroll 1
  for (int dt = -2; dt <= 2; ++dt) {
    if (full) {  // all 50 gathers of the frame in flight, then the arithmetic
      uint64_t tv[25], sv[25];
#pragma unroll
      for (int dy = -2; dy <= 2; ++dy) {
        int ro = dt * a.g.HW + dy * a.g.W;
#pragma unroll
        for (int dx = -2; dx <= 2; ++dx) {
          tv[(dy + 2) * 5 + dx + 2] = __ldg(v + (p + ro + dx));
          sv[(dy + 2) * 5 + dx + 2] = __ldg(v + (q + ro + dx));
        }
      }
#pragma unroll
      for (int k = 0; k < 25; ++k) {
        uint32_t dc = __vabsdiffu4((uint32_t)tv[k], (uint32_t)sv[k]);
        uint32_t dx_ = __vabsdiffu4((uint32_t)(tv[k] >> 32), (uint32_t)(sv[k] >> 32));
        accc = __dp4a(dc, dc, accc);
        acct = __dp4a(dx_, dx_, acct);
        if (SUMS) {  // R42: the target patch's channel sums on the way (evaluate)
          uint32_t(&S)[5] = *reinterpret_cast<uint32_t(*)[5]>(psums);
          vox_add(tv[k], S);
        }
      }
    } else {  // border target: one branch-guarded voxel at a time (rare)
#pragma unroll
      for (int dy = -2; dy <= 2; ++dy) {
        int ro = dt * a.g.HW + dy * a.g.W;
        const unsigned long long* tr = v + (p + ro);
        const unsigned long long* sr = v + (q + ro);
#pragma unroll
        for (int dx = -2; dx <= 2; ++dx) {
          if (!inside(a.g, px + dx, py + dy, pt + dt)) continue;
          if (kb >= 0 && !(a.layer[p + ro + dx] < kb)) continue;
          uint64_t t = __ldg(tr + dx), s = __ldg(sr + dx);
          VINP_ACC(t, s)
        }
      }
    }
    if (ABORT) {
      uint32_t part = 4u * accc + (uint32_t)lambda * acct;
      if (part >= thr) alive = false;
      if (!__any_sync(__activemask(), alive)) break;
      if (!alive) break;
    }
  }
  return 4u * accc + (uint32_t)lambda * acct;
}

// ------------------------------------------------------------------ a5: evaluate
__global__ void __launch_bounds__(256) k_evaluate(LevelArgs a, uint64_t* __restrict__ ee,
                                                  uint8_t* __restrict__ en, uint8_t* __restrict__ es,
                                                  int lambda, int kb, int only_layer, int32_t b,
                                                  int32_t e, const int32_t* __restrict__ list,
                                                  unsigned long long* counter, Mirror mo) {
  int idx = b + blockIdx.x * blockDim.x + threadIdx.x;
  bool act = idx < e;
  int s = act ? (list ? __ldg(list + idx) : idx) : 0;
  if (act && es) put_u8(es, mo.st, mo.n, s, 0);  // pass 0 of the ANN search (R41)
  int p = act ? __ldg(a.targets + s) : 0;
  act = act && (only_layer < 0 || a.layer[p] == only_layer);
  unsigned cnt = 0;
  if (act) {
    int px, py, pt;
    decode(a.g, p, px, py, pt);
    int q = e_q(ee[s]);
    bool full = kb < 0 && px >= 2 && px < a.g.W - 2 && py >= 2 && py < a.g.H - 2 && pt >= 2 && pt < a.g.T - 2;
    bool alive = true;
    uint32_t S[5] = {0, 0, 0, 0, 0};
    uint32_t D = a.psum ? thread_ssd<false, true>(a, p, px, py, pt, q, lambda, kb, full, 0, alive, S)
                        : thread_ssd<false>(a, p, px, py, pt, q, lambda, kb, full, 0, alive);
    // R42: a full target patch leaves its channel sums on the u this search runs on
    if (a.psum && full) const_cast<uint4*>(a.psum)[p] = psum_pack(S);
    int n = 0;
    if (full) {
      n = 125;
    } else {
      for (int dt = -2; dt <= 2; ++dt)
        for (int dy = -2; dy <= 2; ++dy)
          for (int dx = -2; dx <= 2; ++dx)
            if (inside(a.g, px + dx, py + dy, pt + dt) &&
                (kb < 0 || a.layer[p + dt * a.g.HW + dy * a.g.W + dx] < kb))
              ++n;
    }
    put_e(ee, mo, s, pack_e(D, q));
    put_u8(en, mo.nn, mo.n, s, (uint8_t)n);
    cnt = 1;
  }
  cnt = __reduce_add_sync(kFull, cnt);
  if ((threadIdx.x & 31) == 0) flush_count(counter, cnt);
}

// ------------------------------------------------------------------ R42: patch sums
// psum[p] = the five channel sums of vox over N_p (u16 each: <= 125 * 255), for voxels whose whole
// patch lies in Omega.  With them 125 D(p, q) >= 4 |dS_rgb|^2 + lambda |dS_T|^2 (Cauchy-Schwarz
// over the 125 voxels), the exact lower bound random search tests before reading any patch row.
// every voxel: one thread per (x, y) column marching along t with a ring of the last five
// per-frame 5x5 sums (25 gathers per voxel instead of 125)
__global__ void __launch_bounds__(128) k_patch_sums_dense(LevelArgs a, uint4* __restrict__ psum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.g.HW) return;
  const int y = i / a.g.W, x = i - y * a.g.W;
  const bool ok = x >= 2 && x < a.g.W - 2 && y >= 2 && y < a.g.H - 2;
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox);
  uint32_t f0[5] = {0, 0, 0, 0, 0}, f1[5] = {0, 0, 0, 0, 0}, f2[5] = {0, 0, 0, 0, 0}, f3[5] = {0, 0, 0, 0, 0};
  uint32_t S[5] = {0, 0, 0, 0, 0};  // sum of the ring
  for (int t = 0; t < a.g.T; ++t) {
    uint32_t n[5] = {0, 0, 0, 0, 0};
    if (ok) {
      const unsigned long long* c = v + (int64_t)t * a.g.HW + i;
#pragma unroll
      for (int dy = -2; dy <= 2; ++dy)
#pragma unroll
        for (int dx = -2; dx <= 2; ++dx) vox_add(__ldg(c + dy * a.g.W + dx), n);
    }
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      S[c] += n[c];  // ring = frames t-4 .. t, centre t-2
    }
    if (t >= 4) psum[(int64_t)(t - 2) * a.g.HW + i] = ok ? psum_pack(S) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      S[c] -= f0[c];
      f0[c] = f1[c];
      f1[c] = f2[c];
      f2[c] = f3[c];
      f3[c] = n[c];
    }
  }
  // centres without a full patch along t
  for (int t = 0; t < a.g.T; ++t)
    if (t < 2 || t >= a.g.T - 2) psum[(int64_t)t * a.g.HW + i] = make_uint4(0, 0, 0, 0);
}

// the targets of slots [b, e) on the current u (thread per target, x-adjacent lanes)
__global__ void __launch_bounds__(128) k_patch_sums_targets(LevelArgs a, uint4* __restrict__ psum, int32_t b,
                                                            int32_t e) {
  const int s = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= e) return;
  const int p = __ldg(a.targets + s);
  int px, py, pt;
  decode(a.g, p, px, py, pt);
  if (!interior(a.g, px, py, pt)) return;
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox) + p;
  uint32_t S[5] = {0, 0, 0, 0, 0};
#pragma unroll 1
  for (int dt = -2; dt <= 2; ++dt)
#pragma unroll
    for (int dy = -2; dy <= 2; ++dy)
#pragma unroll
      for (int dx = -2; dx <= 2; ++dx) vox_add(__ldg(v + dt * a.g.HW + dy * a.g.W + dx), S);
  psum[p] = psum_pack(S);
}

// 4 |dS_rgb|^2 + lambda |dS_T|^2 >= 125 D_incumbent: the candidate cannot strictly improve
__device__ __forceinline__ bool lb_reject(const uint4 sp, const uint4 sq, int lambda, uint64_t thr) {
  const int dR = (int)(sp.x & 0xffffu) - (int)(sq.x & 0xffffu), dG = (int)(sp.x >> 16) - (int)(sq.x >> 16);
  const int dB = (int)(sp.y & 0xffffu) - (int)(sq.y & 0xffffu), dX = (int)(sp.y >> 16) - (int)(sq.y >> 16);
  const int dY = (int)(sp.z & 0xffffu) - (int)(sq.z & 0xffffu);
  const uint32_t c = (uint32_t)(dR * dR) + (uint32_t)(dG * dG) + (uint32_t)(dB * dB);  // <= 3 * 31875^2 < 2^32
  const uint64_t t = (uint64_t)(uint32_t)(dX * dX) + (uint32_t)(dY * dY);
  return 4ull * c + (uint64_t)lambda * t >= thr;
}

// ------------------------------------------------------------------ R41: targets with a live proposal
// Before an R41-active pass over the slots [b, e) of a level (lv->active): every target of [b, e) copies its
// entry and stamp to the output buffer, and every target whose entry changed since the previous
// pass with the same (step, sign) (stamp >= since) appends the targets that read it in this pass,
// p - sign*step*e_axis (both signs for sign = 0), in a bitmap; k_prop_compact turns it into a list.
// Only the listed targets can have a non-stale proposal; the propagation kernel then runs over the
// list alone.  Workspace words: [0] the list length (zeroed by the launcher), [8 ..) the bitmap
// (all zero between passes), then the list.
__host__ __device__ inline size_t active_bitmap_words(int32_t n) { return ((size_t)n + 31) / 32; }
__global__ void __launch_bounds__(256) k_prop_mark(LevelArgs a, const uint64_t* __restrict__ ein,
                                                   uint64_t* __restrict__ eout, const uint8_t* __restrict__ sin,
                                                   uint8_t* __restrict__ sout, uint32_t* __restrict__ ws, int step,
                                                   int sign, int since, int32_t b, int32_t e, int32_t n) {
  // every target's stamp is looked at (a changed entry outside the slab [b, e) is read by targets
  // inside it; the caller has exchanged those rows), entries are copied and readers flagged in
  // [b, e) only
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint8_t st = __ldg(sin + s);
  if (s >= b && s < e) {
    eout[s] = __ldg(reinterpret_cast<const unsigned long long*>(ein) + s);
    sout[s] = st;
  }
  if ((int)st < since) return;
  uint32_t* bitmap = ws + 8;
  const int p = __ldg(a.targets + s);
  int px, py, pt;
  decode(a.g, p, px, py, pt);
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const int sg = c < 3 ? -1 : 1;  // reader = p - sg' * step * e_axis for each neighbour sign sg' of the pass
    if (sign != 0 && sg != -sign) continue;
    const int ax = c % 3;
    const int x = px + (ax == 0 ? sg * step : 0), y = py + (ax == 1 ? sg * step : 0), t = pt + (ax == 2 ? sg * step : 0);
    if (!inside(a.g, x, y, t)) continue;
    const int r = __ldg(a.slot + lin(a.g, x, y, t));
    if (r < b || r >= e) continue;  // (-1: not a target)
    atomicOr(bitmap + (r >> 5), 1u << (r & 31));
  }
}

// the flagged slots in ascending order within each group of 1024 (x-adjacent targets stay adjacent,
// so the pass's gathers coalesce as in the whole-range kernel); clears the bitmap
__global__ void __launch_bounds__(256) k_prop_compact(uint32_t* __restrict__ ws, int32_t n) {
  const size_t words = active_bitmap_words(n);
  const size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t* bitmap = ws + 8;
  int32_t* list = reinterpret_cast<int32_t*>(bitmap + words);
  uint32_t word = w < words ? bitmap[w] : 0u;
  if (word) bitmap[w] = 0u;
  const int lane = threadIdx.x & 31;
  const int c = __popc(word);
  int incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;
  }
  const int total = __shfl_sync(kFull, incl, 31);
  if (total == 0) return;
  uint32_t base = 0;
  if (lane == 31) base = atomicAdd(ws, (uint32_t)total);
  base = __shfl_sync(kFull, base, 31);
  uint32_t off = base + incl - c;
  while (word) {
    const int bpos = __ffs(word) - 1;
    word &= word - 1u;
    list[off++] = (int32_t)(w * 32 + bpos);
  }
}

// ------------------------------------------------------------------ a6: propagation pass
// Lane = target (thread-per-target, coherent candidates).  Candidates of rank 1..3 are evaluated
// one rank at a time by all lanes that have one, each against the running best of its own target
// (strict improvement in rank order, R25).
// NCMAX 3: one sign per pass; 6: both signs (sign = 0).  LIGHT: every warp takes the column-group
// path (no frame-major per-lane path), compiled for more resident warps — the passes of an ANN
// search after the first same-(step, sign) pass, where the R41 skip leaves few live candidates and
// the candidate-generation latency chain is the cost.
template <int NCMAX, bool LIGHT>
__global__ void __launch_bounds__(LIGHT ? 128 : 256, LIGHT ? VINP_PROP_LIGHT_MINB : VINP_PROP_MINB) k_propagate(LevelArgs a, const uint64_t* __restrict__ ein,
                                                   uint64_t* __restrict__ eout,
                                                   const uint8_t* __restrict__ sin,
                                                   uint8_t* __restrict__ sout, int lambda, int step,
                                                   int sign, int kb, int only_layer, int32_t b,
                                                   int32_t e, int pass, int since,
                                                   const int32_t* __restrict__ list,
                                                   unsigned long long* counter, Mirror mo,
                                                   uint32_t* __restrict__ active) {
  if (active) {
    // the pass runs over the list k_prop_mark built (the entries of the other targets are already
    // copied): [b, e) becomes [0, list length)
    b = 0;
    e = (int32_t)active[0];
    list = reinterpret_cast<const int32_t*>(active + 8 + active_bitmap_words(a.n_targets));
    if ((int)(blockIdx.x * blockDim.x) >= e) return;
  }
  int idx = b + blockIdx.x * blockDim.x + threadIdx.x;
  bool have = idx < e;
  int s = have ? (list ? __ldg(list + idx) : idx) : 0;
  int p = have ? __ldg(a.targets + s) : 0;
  uint64_t inc = have ? __ldg(reinterpret_cast<const unsigned long long*>(ein) + s) : 0ull;
  bool act = have && (only_layer < 0 || a.layer[p] == only_layer);
  // sign = +1 / -1: neighbours p + sign*step*e_{x,y,t}; sign = 0 ("both"): p - step*e_{x,y,t}
  // then p + step*e_{x,y,t} (rank order 1..6)
  const int nc = NCMAX;
  int q[NCMAX];
  bool stl[NCMAX];
#pragma unroll
  for (int c = 0; c < NCMAX; ++c) {
    q[c] = -1;
    stl[c] = false;
  }
  int px = 0, py = 0, pt = 0;
  int q0 = e_q(inc);
  unsigned nstale = 0, nlb = 0;
  if (act) {
    decode(a.g, p, px, py, pt);
    // candidate generation in three branch-free rounds, every load of a round in flight together
    // (out-of-range entries read a safe address and are masked): neighbour slots; their NNF
    // entries and stamps; the D~ flag of each proposed source q = p + (src - r)
    int ox[NCMAX], oy[NCMAX], ot[NCMAX], ra[NCMAX];
    bool ok[NCMAX];
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) {
      const int sg = sign != 0 ? sign : (c < 3 ? -1 : 1);
      const int ax = c % 3;
      ox[c] = ax == 0 ? sg * step : 0;
      oy[c] = ax == 1 ? sg * step : 0;
      ot[c] = ax == 2 ? sg * step : 0;
      ok[c] = c < nc && inside(a.g, px + ox[c], py + oy[c], pt + ot[c]);
      ra[c] = ok[c] ? lin(a.g, px + ox[c], py + oy[c], pt + ot[c]) : p;
    }
    int rs[NCMAX];
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) rs[c] = c < nc ? __ldg(a.slot + ra[c]) : -1;
    uint64_t en[NCMAX];
    uint32_t sn[NCMAX];
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) {
      ok[c] = ok[c] && rs[c] >= 0;
      const int r = ok[c] ? rs[c] : s;
      en[c] = c < nc ? __ldg(reinterpret_cast<const unsigned long long*>(ein) + r) : 0ull;
      sn[c] = (c < nc && since > 0) ? __ldg(sin + r) : 255u;
    }
    int qa[NCMAX];
    uint32_t fl[NCMAX];
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) {
      int sx, sy, st;
      decode(a.g, e_q(en[c]), sx, sy, st);
      const int qx = sx - ox[c], qy = sy - oy[c], qt = st - ot[c];  // q = p + (src - r)
      ok[c] = ok[c] && inside(a.g, qx, qy, qt);
      qa[c] = ok[c] ? lin(a.g, qx, qy, qt) : p;
      fl[c] = c < nc ? __ldg(a.flags + qa[c]) : 0u;
    }
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) {
      if (ok[c] && (fl[c] & 2)) q[c] = qa[c];
      stl[c] = sn[c] < (uint32_t)since;  // R41: unchanged since pass `since` (since = 0: never)
    }
    // keep a candidate only if it differs from the incumbent and every earlier valid candidate
#pragma unroll
    for (int c = NCMAX - 1; c >= 0; --c) {
      bool dup = q[c] == q0;
#pragma unroll
      for (int c2 = 0; c2 < c; ++c2) dup |= (q[c2] == q[c]);
      if (dup) q[c] = -1;
    }
    // then drop the stale survivors (R41): they cannot beat the incumbent
#pragma unroll
    for (int c = 0; c < NCMAX; ++c)
      if (q[c] >= 0 && stl[c]) {
        q[c] = -1;
        ++nstale;
      }
#if VINP_PROP_LB
    // R42: then the candidates whose patch-sum lower bound reaches the incumbent's D (every one if
    // that D is 0): tested against the incumbent, hence counted, but no patch row is read
    if (a.psum && kb < 0 && interior(a.g, px, py, pt)) {
      bool any = false;
#pragma unroll
      for (int c = 0; c < NCMAX; ++c) any |= q[c] >= 0;
      const uint64_t thr = 125ull * e_D(inc);
      if (any && thr == 0) {
#pragma unroll
        for (int c = 0; c < NCMAX; ++c)
          if (q[c] >= 0) {
            q[c] = -1;
            ++nlb;
          }
      } else if (!LIGHT && any) {  // (the R41-active passes keep only the free D = 0 test: A/B)
        const uint4 sp = __ldg(a.psum + p);
        uint4 sq[NCMAX];
#pragma unroll
        for (int c = 0; c < NCMAX; ++c) sq[c] = __ldg(a.psum + (q[c] >= 0 ? q[c] : p));
#pragma unroll
        for (int c = 0; c < NCMAX; ++c)
          if (q[c] >= 0 && lb_reject(sp, sq[c], lambda, thr)) {
            q[c] = -1;
            ++nlb;
          }
      }
    }
#endif
  }
  // compact this lane's candidates to the front (rank order kept), so that the warp runs the
  // SSD loop once per candidate *slot* rather than once per neighbour rank any lane has
  int cq[NCMAX];
  int ncand = 0;
#pragma unroll
  for (int c = 0; c < NCMAX; ++c) cq[c] = -1;
#pragma unroll
  for (int c = 0; c < NCMAX; ++c) {
    if (act && q[c] >= 0) {
#pragma unroll
      for (int d = 0; d < NCMAX; ++d)
        if (d == ncand) cq[d] = q[c];
      ++ncand;
    }
  }
  uint32_t bestD = e_D(inc);
  int bestq = q0;
  unsigned cnt = nlb;  // R42 rejections are patch-updates too
#if VINP_PROP_SPARSE > 0
  {
    // Sparse warp (few live candidates, typical once the R41 skip has removed the stale ones):
    // the warp's (candidate, owner) pairs are evaluated by 5-lane column groups, six at a time,
    // instead of by their owner lanes with the other lanes idle.  Same rank order, same exact
    // early abort, same result.
    int incl = ncand;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(kFull, incl, d);
      if ((threadIdx.x & 31) >= d) incl += y;
    }
    const int P = __shfl_sync(kFull, incl, 31);
    if (LIGHT || P <= VINP_PROP_SPARSE) {  // warp-uniform
      constexpr int kCap = LIGHT ? 32 * NCMAX : VINP_PROP_SPARSE;
      __shared__ int2 s_pairs[(LIGHT ? 128 : 256) / 32][kCap];
      int2* pairs = s_pairs[threadIdx.x >> 5];
#pragma unroll
      for (int c = 0; c < NCMAX; ++c)
        if (c < ncand) pairs[incl - ncand + c] = make_int2(cq[c], (c << 5) | (threadIdx.x & 31));
      __syncwarp();
      group_eval(a, pairs, P, threadIdx.x & 31, p, px, py, pt, lambda, bestD, bestq);
      if (have) {
        put_e(eout, mo, s, pack_e(bestD, bestq));
        if (sout) put_u8(sout, mo.st, mo.n, s, bestq != q0 ? (uint8_t)pass : __ldg(sin + s));
      }
      nstale = active ? 0u : __reduce_add_sync(kFull, nstale);  // no stale count with `active`
      cnt = __reduce_add_sync(kFull, cnt);
      if ((threadIdx.x & 31) == 0) {
        flush_count(counter, (unsigned)P + cnt);
        if (counter && nstale) flush_count(counter + 1, nstale);
      }
      return;
    }
  }
#endif
  if constexpr (!LIGHT) {
  bool full = act && kb < 0 && px >= 2 && px < a.g.W - 2 && py >= 2 && py < a.g.H - 2 && pt >= 2 &&
              pt < a.g.T - 2;
  bool allfull = __all_sync(kFull, full || !act);
#if VINP_PROP_FRAME_MAJOR
  if (allfull) {
    // Row-major over the patch, all of this lane's candidates per target row: each target row (5
    // coalesced 8-byte gathers) is loaded once and compared with the same row of every live
    // candidate, instead of once per candidate.  A candidate is dropped after a frame once its
    // partial sum reaches the incumbent's D (it can then never be accepted: exact, R35); the
    // survivors are applied in rank order with strict improvement (R25).
    const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox);
    uint32_t accc[NCMAX], acct[NCMAX];
    unsigned alive = 0;
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) {
      accc[c] = acct[c] = 0;
      if (c < ncand) alive |= 1u << c;
    }
    cnt += ncand;
    const uint32_t thr = bestD;
#pragma unroll 1
    for (int dt = -2; dt <= 2; ++dt) {
      if (!__any_sync(kFull, alive != 0)) break;
#pragma unroll
      for (int dy = -2; dy <= 2; ++dy) {
        const int ro = dt * a.g.HW + dy * a.g.W;
        uint64_t tv[5];
#pragma unroll
        for (int dx = -2; dx <= 2; ++dx) tv[dx + 2] = alive ? __ldg(v + (p + ro + dx)) : 0ull;
#pragma unroll
        for (int c = 0; c < NCMAX; ++c) {
          if (!((alive >> c) & 1)) continue;
          uint64_t sv[5];
#pragma unroll
          for (int dx = -2; dx <= 2; ++dx) sv[dx + 2] = __ldg(v + (cq[c] + ro + dx));
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            uint32_t dc = __vabsdiffu4((uint32_t)tv[k], (uint32_t)sv[k]);
            uint32_t dx_ = __vabsdiffu4((uint32_t)(tv[k] >> 32), (uint32_t)(sv[k] >> 32));
            accc[c] = __dp4a(dc, dc, accc[c]);
            acct[c] = __dp4a(dx_, dx_, acct[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NCMAX; ++c)
        if (4u * accc[c] + (uint32_t)lambda * acct[c] >= thr) alive &= ~(1u << c);
    }
#pragma unroll
    for (int c = 0; c < NCMAX; ++c) {
      const uint32_t D = 4u * accc[c] + (uint32_t)lambda * acct[c];
      if (((alive >> c) & 1) && D < bestD) {
        bestD = D;
        bestq = cq[c];
      }
    }
    if (have) {
      put_e(eout, mo, s, pack_e(bestD, bestq));
      if (sout) put_u8(sout, mo.st, mo.n, s, bestq != q0 ? (uint8_t)pass : __ldg(sin + s));
    }
    cnt = __reduce_add_sync(kFull, cnt);
    nstale = __reduce_add_sync(kFull, nstale);
    if ((threadIdx.x & 31) == 0) {
      flush_count(counter, cnt);
      if (counter && nstale) flush_count(counter + 1, nstale);
    }
    return;
  }
#endif
#pragma unroll
  for (int c = 0; c < NCMAX; ++c) {
    bool mine = c < ncand;
    if (!__any_sync(kFull, mine)) break;
    if (mine) {
      bool alive = true;
      uint32_t D = allfull ? thread_ssd<true>(a, p, px, py, pt, cq[c], lambda, kb, true, bestD, alive)
                           : thread_ssd<true>(a, p, px, py, pt, cq[c], lambda, kb, full, bestD, alive);
      if (alive && D < bestD) {
        bestD = D;
        bestq = cq[c];
      }
      ++cnt;
    }
  }
  if (have) {
    put_e(eout, mo, s, pack_e(bestD, bestq));
    if (sout) put_u8(sout, mo.st, mo.n, s, bestq != q0 ? (uint8_t)pass : __ldg(sin + s));
  }
  cnt = __reduce_add_sync(kFull, cnt);
  nstale = __reduce_add_sync(kFull, nstale);
  if ((threadIdx.x & 31) == 0) {
    flush_count(counter, cnt);
    if (counter && nstale) flush_count(counter + 1, nstale);
  }
  }
}

// Warp-per-target patch (onion passes): lane l owns the voxels k = l + 32 j (j < 4, k < 125) of
// N_p; a voxel outside Omega or K contributes nothing (its target word is zeroed and its source
// gather skipped).  load() issues the gathers, mask() consumes the layer bytes.
struct WideTarget {
  uint64_t tv[4];
  uint8_t lay[4];
  int off[4];
  bool ok[4];
  __device__ __forceinline__ void load(const LevelArgs& a, int p, int px, int py, int pt, int lane) {
    const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = lane + 32 * j;
      const int dt = k / 25 - 2, dy = (k % 25) / 5 - 2, dx = k % 5 - 2;
      off[j] = dt * a.g.HW + dy * a.g.W + dx;
      ok[j] = k < 125 && inside(a.g, px + dx, py + dy, pt + dt);
      lay[j] = ok[j] ? a.layer[p + off[j]] : (uint8_t)255;
      tv[j] = ok[j] ? __ldg(v + (p + off[j])) : 0ull;
    }
  }
  __device__ __forceinline__ void mask(int kb) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ok[j] = ok[j] && (kb < 0 || (int)lay[j] < kb);
      if (!ok[j]) tv[j] = 0ull;
    }
  }
  // this lane's share of D(p, q) (Eq. 9, R24 integer form); q in D~, so every gather is in bounds
  __device__ __forceinline__ uint32_t part(const unsigned long long* v, int q, int lambda) const {
    uint64_t sv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) sv[j] = ok[j] ? __ldg(v + (q + off[j])) : 0ull;
    uint32_t accc = 0, acct = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) VINP_ACC(tv[j], sv[j])
    return 4u * accc + (uint32_t)lambda * acct;
  }
};

#ifndef VINP_WIDE_BLOCK
#define VINP_WIDE_BLOCK 64
#endif
// Onion (K-restricted) propagation pass, warp per target.  An onion layer holds a few hundred to
// a few ten thousand targets, so a thread-per-target pass runs as one latency chain per lane
// (candidate generation, then per frame layer bytes -> predicated voxels, up to 15 frames): it
// measured ~40 us per launch whatever its size, x 880 launches per c5 step.  Here the 125 voxels of the
// patch are spread over the warp (lane l owns k = l + 32 j), the (up to 6) candidates are
// generated by lanes 0..nc-1 in parallel, and all candidate gathers are issued at once, so the
// chain is ~8 round trips.  No early abort: a candidate is kept iff D < best in rank order (R25),
// the same decision the aborting pass takes; counts one patch-update per evaluated candidate.
__global__ void __launch_bounds__(VINP_WIDE_BLOCK) k_propagate_wide(
    LevelArgs a, const uint64_t* __restrict__ ein, uint64_t* __restrict__ eout,
    const uint8_t* __restrict__ sin, uint8_t* __restrict__ sout, int lambda, int step, int sign,
    int kb, int only_layer, int32_t b, int32_t e, int pass, int since,
    const int32_t* __restrict__ list, unsigned long long* counter, Mirror mo) {
  const int lane = threadIdx.x & 31;
  const int idx = b + (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  if (idx >= e) return;  // warp-uniform
  const int s = list ? __ldg(list + idx) : idx;
  const int p = __ldg(a.targets + s);
  const uint64_t inc = __ldg(reinterpret_cast<const unsigned long long*>(ein) + s);
  // a filtered full-range launch (per-pass path): most warps leave here.  With a layer list
  // (vinp_onion_peel) every target is in the layer, and the test waits until the end
  if (!list && only_layer >= 0 && a.layer[p] != only_layer) {
    if (lane == 0) {
      put_e(eout, mo, s, inc);
      if (sout) put_u8(sout, mo.st, mo.n, s, sin[s]);
    }
    return;
  }
  const bool act = only_layer < 0 || a.layer[p] == only_layer;  // used at the end: no stall here
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox);
  int px, py, pt;
  decode(a.g, p, px, py, pt);
  // the target side first (independent of the candidates, in flight during their generation)
  WideTarget w;
  w.load(a, p, px, py, pt, lane);
  const int nc = sign == 0 ? 6 : 3;
  // candidate c on lane c (neighbour shift -> its NNF entry -> q = p + (src - r) -> q in D~?)
  int myq = -1;
  bool mystl = false;
  if (lane < nc) {
    const int c = lane;
    const int sg = sign != 0 ? sign : (c < 3 ? -1 : 1);
    const int ax = c % 3;
    const int ox = ax == 0 ? sg * step : 0, oy = ax == 1 ? sg * step : 0, ot = ax == 2 ? sg * step : 0;
    const int rx = px + ox, ry = py + oy, rt = pt + ot;
    if (inside(a.g, rx, ry, rt)) {
      const int rs = __ldg(a.slot + lin(a.g, rx, ry, rt));
      if (rs >= 0) {
        const int src = e_q(__ldg(reinterpret_cast<const unsigned long long*>(ein) + rs));
        if (since > 0) mystl = __ldg(sin + rs) < since;  // R41
        int sx, sy, st;
        decode(a.g, src, sx, sy, st);
        const int qx = sx - ox, qy = sy - oy, qt = st - ot;
        if (is_source(a.g, a.flags, qx, qy, qt)) myq = lin(a.g, qx, qy, qt);
      }
    }
  }
  w.mask(kb);
  // de-duplicate exactly as the thread pass: drop a candidate equal to the incumbent or to an
  // earlier candidate
  const int q0 = e_q(inc);
  int q[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) q[c] = __shfl_sync(kFull, myq, c);
  const unsigned stlm = __ballot_sync(kFull, mystl);
  bool keep[6];
  unsigned nstale = 0;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    bool dup = !act || c >= nc || q[c] < 0 || q[c] == q0;
#pragma unroll
    for (int c2 = 0; c2 < c; ++c2) dup |= (q[c2] == q[c]);
    keep[c] = !dup;
    if (keep[c] && ((stlm >> c) & 1)) {  // R41: stale, cannot win
      keep[c] = false;
      ++nstale;
    }
  }
  // all candidate gathers in flight together (q in D~: its whole patch lies in the volume)
  uint32_t part[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) part[c] = keep[c] ? w.part(v, q[c], lambda) : 0u;
  uint32_t bestD = e_D(inc);
  int bestq = q0;
  unsigned cnt = 0;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    if (!keep[c]) continue;  // warp-uniform
    const uint32_t D = __reduce_add_sync(kFull, part[c]);
    if (D < bestD) {
      bestD = D;
      bestq = q[c];
    }
    ++cnt;
  }
  if (lane == 0) {
    put_e(eout, mo, s, pack_e(bestD, bestq));
    if (sout) put_u8(sout, mo.st, mo.n, s, bestq != q0 ? (uint8_t)pass : sin[s]);
    flush_count(counter, cnt);
    if (counter && nstale) flush_count(counter + 1, nstale);
  }
}

// Onion (K-restricted) evaluate, warp per target: D(p, phi(p)) over the voxels of N_p in Omega
// and K (Alg. 3: only known voxels count) and their number n.
__global__ void __launch_bounds__(VINP_WIDE_BLOCK) k_evaluate_wide(LevelArgs a, uint64_t* __restrict__ ee,
                                                                   uint8_t* __restrict__ en,
                                                                   uint8_t* __restrict__ es, int lambda,
                                                                   int kb, int only_layer, int32_t b,
                                                                   int32_t e, const int32_t* __restrict__ list,
                                                                   unsigned long long* counter, Mirror mo) {
  const int lane = threadIdx.x & 31;
  const int idx = b + (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  if (idx >= e) return;  // warp-uniform
  const int s = list ? __ldg(list + idx) : idx;
  if (es && lane == 0) put_u8(es, mo.st, mo.n, s, 0);  // pass 0 of the ANN search (R41)
  const int p = __ldg(a.targets + s);
  if (only_layer >= 0 && a.layer[p] != only_layer) return;
  int px, py, pt;
  decode(a.g, p, px, py, pt);
  WideTarget w;
  w.load(a, p, px, py, pt, lane);
  const int q = e_q(ee[s]);
  w.mask(kb);
  const uint32_t D = __reduce_add_sync(kFull, w.part(reinterpret_cast<const unsigned long long*>(a.vox), q, lambda));
  const uint32_t n = __reduce_add_sync(kFull, (uint32_t)(w.ok[0] + w.ok[1] + w.ok[2] + w.ok[3]));
  if (lane == 0) {
    put_e(ee, mo, s, pack_e(D, q));
    put_u8(en, mo.nn, mo.n, s, (uint8_t)n);
    flush_count(counter, 1);
  }
}

// ------------------------------------------------------------------ a7: random search pass
struct Radii {
  double R[32];
  int M;
};

template <int NC, int WPB, int TPW>
__global__ void __launch_bounds__(32 * WPB, VINP_MINB * 8 / WPB) k_random_search(
    LevelArgs a, const uint64_t* __restrict__ ein, uint64_t* __restrict__ eout,
    const uint8_t* __restrict__ sin, uint8_t* __restrict__ sout, int lambda, Radii rad,
    uint64_t seed, uint32_t oc, int pm_iter, int only_layer, int32_t b, int32_t e, int pass,
    const int32_t* __restrict__ list, unsigned long long* counter, Mirror mo) {
  // TPW targets per warp (32; 8 for small launches, so that more warps share
  // the pair evaluations — the result does not depend on it)
  int lane = threadIdx.x & 31;
  int i0 = b + (blockIdx.x * WPB + (threadIdx.x >> 5)) * TPW;
  if (i0 >= e) return;
  int idx = i0 + lane;
  bool have = (TPW == 32 || lane < TPW) && idx < e;
  int s = have ? (list ? __ldg(list + idx) : idx) : 0;
  int p = have ? __ldg(a.targets + s) : 0;
  uint64_t inc = have ? __ldg(reinterpret_cast<const unsigned long long*>(ein) + s) : 0ull;
  bool act = have && (only_layer < 0 || a.layer[p] == only_layer);
  __shared__ int s_cand[WPB][NC * 32];
  __shared__ int2 s_pairs[WPB][NC * 32];
  int* cand = s_cand[threadIdx.x >> 5];
  int2* pairs = s_pairs[threadIdx.x >> 5];
  int nc = 0;
  unsigned rej = 0;  // R42: bit j = candidate j rejected by the lower bound
  int px = 0, py = 0, pt = 0;
  if (act) {
    decode(a.g, p, px, py, pt);
    int q0 = e_q(inc);
    int q0x, q0y, q0t;
    decode(a.g, q0, q0x, q0y, q0t);
#if VINP_RS_GEN_CHUNK > 1
    // candidates i + 1 of Eq. 3 in chunks: the Philox draws of a chunk, then its D~ flag loads in
    // flight together, then the de-duplication in rank order
    for (int i0 = 0; i0 < rad.M; i0 += VINP_RS_GEN_CHUNK) {
      int qv[VINP_RS_GEN_CHUNK];
#pragma unroll
      for (int j = 0; j < VINP_RS_GEN_CHUNK; ++j) {
        const int i = min(i0 + j, rad.M - 1);
        uint4 u = draw((uint32_t)p, (uint32_t)pm_iter, a.level, kStreamRS, i + 1, oc, seed);
        double R = rad.R[i];
        int ox = (int)floor(__dmul_rn(R, __dmul_rn((double)u.x - 2147483648.0, 4.656612873077392578125e-10)));
        int oy = (int)floor(__dmul_rn(R, __dmul_rn((double)u.y - 2147483648.0, 4.656612873077392578125e-10)));
        int ot = (int)floor(__dmul_rn(R, __dmul_rn((double)u.z - 2147483648.0, 4.656612873077392578125e-10)));
        int qx = q0x + ox, qy = q0y + oy, qt = q0t + ot;
        qv[j] = (i0 + j < rad.M && inside(a.g, qx, qy, qt)) ? lin(a.g, qx, qy, qt) : -1;
      }
      uint32_t fl[VINP_RS_GEN_CHUNK];
#pragma unroll
      for (int j = 0; j < VINP_RS_GEN_CHUNK; ++j) fl[j] = __ldg(a.flags + (qv[j] >= 0 ? qv[j] : p));
#pragma unroll
      for (int j = 0; j < VINP_RS_GEN_CHUNK; ++j) {
        if (qv[j] >= 0 && (fl[j] & 2)) {
          const int qq = qv[j];
          bool dup = qq == q0;
          for (int k = 0; k < nc; ++k) dup |= (cand[k * 32 + lane] == qq);
          if (!dup) cand[(nc++) * 32 + lane] = qq;
        }
      }
    }
#else
    for (int i = 0; i < rad.M; ++i) {  // candidate i + 1 of Eq. 3
      uint4 u = draw((uint32_t)p, (uint32_t)pm_iter, a.level, kStreamRS, i + 1, oc, seed);
      double R = rad.R[i];
      int ox = (int)floor(__dmul_rn(R, __dmul_rn((double)u.x - 2147483648.0, 4.656612873077392578125e-10)));
      int oy = (int)floor(__dmul_rn(R, __dmul_rn((double)u.y - 2147483648.0, 4.656612873077392578125e-10)));
      int ot = (int)floor(__dmul_rn(R, __dmul_rn((double)u.z - 2147483648.0, 4.656612873077392578125e-10)));
      int qx = q0x + ox, qy = q0y + oy, qt = q0t + ot;
      if (is_source(a.g, a.flags, qx, qy, qt)) {
        int qq = lin(a.g, qx, qy, qt);
        bool dup = qq == q0;
        for (int j = 0; j < nc; ++j) dup |= (cand[j * 32 + lane] == qq);
        if (!dup) cand[(nc++) * 32 + lane] = qq;
      }
    }
#endif
    // R42: candidates whose patch-sum lower bound already reaches the incumbent's D cannot win;
    // they stay in `cand` (de-duplication, counts) but are not evaluated
    if (a.psum && nc > 0 && interior(a.g, px, py, pt)) {
      const uint64_t thr = 125ull * e_D(inc);
      if (thr == 0) {
        rej = 0xffffffffu;
      } else {
        const uint4 sp = __ldg(a.psum + p);
#pragma unroll 1
        for (int j0 = 0; j0 < nc; j0 += 4) {
          uint4 sq[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) sq[j] = __ldg(a.psum + (j0 + j < nc ? cand[(j0 + j) * 32 + lane] : p));
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j0 + j < nc && lb_reject(sp, sq[j], lambda, thr)) rej |= 1u << (j0 + j);
        }
      }
    }
  }
  // flatten (owner lane, rank) pairs in lane order: the candidates that are left
  const int ns = nc - __popc(rej & (nc >= 32 ? 0xffffffffu : ((1u << nc) - 1u)));
  int incl = ns;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;
  }
  int P = __shfl_sync(kFull, incl, 31);
#if VINP_RS_ORDER == 0
  // lane-major (owner, rank) order
  for (int j = 0, o = incl - ns; j < nc; ++j)
    if (!((rej >> j) & 1u)) pairs[o++] = make_int2(cand[j * 32 + lane], (j << 5) | lane);
#else
  // rank-major: all owners' candidates of one rank together (1: rank 0 first, 2: last rank first),
  // so that a warp iteration's pairs have similar radii; the rank stays the tie key
  {
    int base = 0;
    for (int jr = 0; jr < NC; ++jr) {
      const int j = VINP_RS_ORDER == 1 ? jr : NC - 1 - jr;
      const bool keep = j < nc && !((rej >> j) & 1u);
      const unsigned mk = __ballot_sync(kFull, keep);
      if (keep) pairs[base + __popc(mk & ((1u << lane) - 1u))] = make_int2(cand[j * 32 + lane], (j << 5) | lane);
      base += __popc(mk);
    }
  }
#endif
  __syncwarp();
  uint32_t bestD = e_D(inc);
  int bestq = e_q(inc);
#ifndef VINP_RS_NOEVAL  // (profiling builds time the candidate generation alone)
  group_eval(a, pairs, P, lane, p, px, py, pt, lambda, bestD, bestq);
#endif
  if (have) {
    put_e(eout, mo, s, pack_e(bestD, bestq));
    if (sout) put_u8(sout, mo.st, mo.n, s, bestq != e_q(inc) ? (uint8_t)pass : __ldg(sin + s));
  }
  // rejected candidates count as patch-updates too (R34: tested against the incumbent)
  const unsigned tot = __reduce_add_sync(kFull, (unsigned)nc);
  if (lane == 0) flush_count(counter, tot);
}

// Random search for onion (K-restricted) launches, warp per target: lane i < M draws candidate
// i + 1 of Eq. 3 (Philox, the same draw and fp64 offset arithmetic as above, so the same q), the
// warp de-duplicates (a candidate equal to the incumbent or to an earlier valid one is dropped),
// then evaluates the kept candidates 4 at a time with every gather of a batch in flight and
// applies them in rank order with strict improvement (R25).
__global__ void __launch_bounds__(VINP_WIDE_BLOCK) k_random_search_wide(
    LevelArgs a, const uint64_t* __restrict__ ein, uint64_t* __restrict__ eout,
    const uint8_t* __restrict__ sin, uint8_t* __restrict__ sout, int lambda, Radii rad,
    uint64_t seed, uint32_t oc, int pm_iter, int kb, int only_layer, int32_t b, int32_t e, int pass,
    const int32_t* __restrict__ list, unsigned long long* counter, Mirror mo) {
  const int lane = threadIdx.x & 31;
  const int idx = b + (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  if (idx >= e) return;  // warp-uniform
  const int s = list ? __ldg(list + idx) : idx;
  const int p = __ldg(a.targets + s);
  const uint64_t inc = __ldg(reinterpret_cast<const unsigned long long*>(ein) + s);
  if (!list && only_layer >= 0 && a.layer[p] != only_layer) {  // as k_propagate_wide
    if (lane == 0) {
      put_e(eout, mo, s, inc);
      if (sout) put_u8(sout, mo.st, mo.n, s, sin[s]);
    }
    return;
  }
  const bool act = only_layer < 0 || a.layer[p] == only_layer;
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox);
  int px, py, pt;
  decode(a.g, p, px, py, pt);
  WideTarget w;
  w.load(a, p, px, py, pt, lane);
  const int q0 = e_q(inc);
  int myq = -1;
  if (lane < rad.M) {  // candidate i + 1 = lane + 1
    int q0x, q0y, q0t;
    decode(a.g, q0, q0x, q0y, q0t);
    uint4 u = draw((uint32_t)p, (uint32_t)pm_iter, a.level, kStreamRS, lane + 1, oc, seed);
    double R = rad.R[lane];
    int ox = (int)floor(__dmul_rn(R, __dmul_rn((double)u.x - 2147483648.0, 4.656612873077392578125e-10)));
    int oy = (int)floor(__dmul_rn(R, __dmul_rn((double)u.y - 2147483648.0, 4.656612873077392578125e-10)));
    int ot = (int)floor(__dmul_rn(R, __dmul_rn((double)u.z - 2147483648.0, 4.656612873077392578125e-10)));
    int qx = q0x + ox, qy = q0y + oy, qt = q0t + ot;
    if (is_source(a.g, a.flags, qx, qy, qt)) myq = lin(a.g, qx, qy, qt);
  }
  w.mask(kb);
  // keep[i]: valid, not the incumbent, not equal to an earlier valid candidate
  bool keep = act && myq >= 0 && myq != q0;
  for (int i = 0; i < rad.M; ++i) {
    const int qi = __shfl_sync(kFull, myq, i);
    if (i < lane && qi >= 0 && qi == myq) keep = false;
  }
  unsigned km = __ballot_sync(kFull, keep);
  const unsigned cnt = __popc(km);
  uint32_t bestD = e_D(inc);
  int bestq = q0;
  while (km) {  // batches of 4 kept candidates, rank order
    int qb[4];
    uint32_t part[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = km ? __ffs(km) - 1 : -1;
      if (km) km &= km - 1u;
      qb[c] = i >= 0 ? __shfl_sync(kFull, myq, i) : -1;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) part[c] = qb[c] >= 0 ? w.part(v, qb[c], lambda) : 0u;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (qb[c] < 0) break;  // warp-uniform
      const uint32_t D = __reduce_add_sync(kFull, part[c]);
      if (D < bestD) {
        bestD = D;
        bestq = qb[c];
      }
    }
  }
  if (lane == 0) {
    put_e(eout, mo, s, pack_e(bestD, bestq));
    if (sout) put_u8(sout, mo.st, mo.n, s, bestq != q0 ? (uint8_t)pass : sin[s]);
    flush_count(counter, cnt);
  }
}

// ------------------------------------------------------------------ a13: brute force (CUDA cores)
// One block of 8 warps per target; warp w scans sources i = w, w+8, ... in increasing order, 8 at a
// time with all gathers of a 32-voxel chunk in flight, and keeps its first minimum (strict <).
// Exact partial-distance elimination: a source whose partial sum reaches the warp's best so far
// cannot become the (first) minimum.  The block then takes the lexicographic min of (D, i).
__global__ void __launch_bounds__(256) k_brute_force(LevelArgs a, uint64_t* __restrict__ ee,
                                                     uint8_t* __restrict__ en, int lambda, int32_t b,
                                                     int32_t e, const int32_t* __restrict__ list) {
  constexpr int G = 8;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int idx = b + blockIdx.x;
  if (idx >= e) return;
  int s = list ? list[idx] : idx;
  int p = a.targets[s];
  PatchLanes L;
  init_lanes(L, a.g, lane);
  int px, py, pt;
  decode(a.g, p, px, py, pt);
  TargetPatch tp;
  load_target(tp, L, a.g, a.vox, a.layer, -1, p, px, py, pt);
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(a.vox);
  uint32_t bestD = 0xffffffffu;
  int bestI = 0x7fffffff;
  for (int i0 = w; i0 < a.n_sources; i0 += G * kWarpsPerBlock) {
    int q[G];
    uint32_t part[G];
    unsigned alive = 0;
#pragma unroll
    for (int c = 0; c < G; ++c) {
      int i = i0 + c * kWarpsPerBlock;
      bool ok = i < a.n_sources;
      q[c] = ok ? __ldg(a.sources + i) : 0;
      part[c] = 0;
      alive |= (unsigned)ok << c;
    }
    uint32_t thr = bestD;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      if (!alive) break;
      bool m = (tp.mask >> ch) & 1;
      uint64_t sv[G];
#pragma unroll
      for (int c = 0; c < G; ++c) sv[c] = (m && ((alive >> c) & 1)) ? __ldg(v + q[c] + L.off[ch]) : 0ull;
#pragma unroll
      for (int c = 0; c < G; ++c) {
        if ((alive >> c) & 1) {
          uint32_t x = m ? voxel_cost(tp.c[ch], tp.t[ch], sv[c], lambda) : 0u;
          part[c] += __reduce_add_sync(kFull, x);
          if (part[c] >= thr) alive &= ~(1u << c);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < G; ++c)
      if (((alive >> c) & 1) && part[c] < bestD) {
        bestD = part[c];
        bestI = i0 + c * kWarpsPerBlock;
      }
  }
  __shared__ unsigned long long red[kWarpsPerBlock];
  if (lane == 0) red[w] = ((uint64_t)bestD << 32) | (uint32_t)bestI;
  __syncthreads();
  uint32_t n = __reduce_add_sync(kFull, (uint32_t)__popc(tp.mask));
  if (threadIdx.x == 0) {
    uint64_t mn = red[0];
    for (int k = 1; k < kWarpsPerBlock; ++k) mn = min(mn, (uint64_t)red[k]);
    ee[s] = pack_e((uint32_t)(mn >> 32), a.sources[(uint32_t)mn]);
    en[s] = (uint8_t)n;
  }
}

// ------------------------------------------------------------------ test hooks
__global__ void k_patch_ssd(LevelArgs a, const int32_t* __restrict__ P, const int32_t* __restrict__ Q,
                            int64_t n, int lambda, int kb, uint32_t* __restrict__ D,
                            uint8_t* __restrict__ cnt) {
  int lane = threadIdx.x & 31;
  int64_t i = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (i >= n) return;
  PatchLanes L;
  init_lanes(L, a.g, lane);
  int p = P[i];
  int px, py, pt;
  decode(a.g, p, px, py, pt);
  TargetPatch tp;
  load_target(tp, L, a.g, a.vox, a.layer, kb, p, px, py, pt);
  uint32_t d = warp_ssd(tp, L, a.vox, Q[i], lambda);
  uint32_t c = __reduce_add_sync(kFull, (uint32_t)__popc(tp.mask));
  if (lane == 0) {
    D[i] = d;
    cnt[i] = (uint8_t)c;
  }
}

__global__ void k_philox(const uint4* __restrict__ ctr, int64_t n, uint64_t seed,
                         uint4* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = philox(ctr[i], (uint32_t)seed, (uint32_t)(seed >> 32));
}

static vinp_status check_nnf_args(const vinp_level* lv, const char* who, int32_t b, int32_t e,
                                  const vinp_params* prm) {
  vinp_status st = check_level(lv, who);
  if (st) return st;
  if (!prm) { set_error("%s: null params", who); return VINP_E_INVALID; }
  if (prm->lambda < 0 || prm->lambda > 126) {
    set_error("%s: lambda %d outside [0,126]", who, prm->lambda);
    return VINP_E_UNSUPPORTED;
  }
  if (b < 0 || e > lv->n_targets || b > e) {
    set_error("%s: slot range [%d,%d) outside [0,%d)", who, b, e, lv->n_targets);
    return VINP_E_INVALID;
  }
  if (!lv->targets || !lv->slot) { set_error("%s: level lists missing", who); return VINP_E_INVALID; }
  return VINP_OK;
}

static Radii make_radii(const vinp_level* lv, const vinp_params* prm) {
  Radii r{};
  int rmax = prm->rmax > 0 ? prm->rmax : std::max(lv->W, std::max(lv->H, lv->T));
  double R = (double)rmax;
  r.M = 0;
  // the kernels hold at most 32 radii (one per lane in the warp-per-target form); a 33rd radius
  // R_33 >= 1 is refused rather than dropped (the oracle would evaluate it)
  for (int i = 1; i <= 33; ++i) {
    R = R * prm->rho;
    if (!(R >= 1.0)) break;
    if (r.M == 32) { r.M = -1; break; }
    r.R[r.M++] = R;
  }
  return r;
}

}  // namespace vinp

using namespace vinp;

extern "C" {

vinp_status vinp_nnf_init_random(const vinp_level* lv, vinp_nnf* nnf, const vinp_params* prm,
                                 uint32_t outer_code, int32_t b, int32_t e, void* stream) {
  VINP_NVTX();
  vinp_status st = check_nnf_args(lv, "vinp_nnf_init_random", b, e, prm);
  if (st) return st;
  VINP_REQUIRE(nnf && nnf->e && nnf->n, "vinp_nnf_init_random: null nnf");
  if (lv->n_sources <= 0) {
    set_error("vinp_nnf_init_random: D~ is empty at level %d", lv->level);
    return VINP_E_NO_SOURCE;
  }
  if (e > b) {
    k_init_random<<<nblk(e - b, 256), 256, 0, S(stream)>>>(args_of(lv), nnf->e, nnf->n, prm->seed,
                                                           outer_code, b, e);
    count_launch();
  }
  return check_launch("vinp_nnf_init_random");
}

vinp_status vinp_nnf_upsample(const vinp_level* coarse, const vinp_nnf* cn, const vinp_level* fine,
                              vinp_nnf* fn, const vinp_params* prm, int32_t b, int32_t e,
                              void* stream) {
  VINP_NVTX();
  vinp_status st = check_nnf_args(fine, "vinp_nnf_upsample", b, e, prm);
  if (st) return st;
  st = check_level(coarse, "vinp_nnf_upsample(coarse)");
  if (st) return st;
  VINP_REQUIRE(cn && cn->e && fn && fn->e && fn->n && coarse->slot, "vinp_nnf_upsample: null nnf");
  VINP_REQUIRE(coarse->T == fine->T && coarse->W == (fine->W + 1) / 2 && coarse->H == (fine->H + 1) / 2,
               "vinp_nnf_upsample: coarse dims must be ceil(fine/2)");
  if (fine->n_sources <= 0) {
    set_error("vinp_nnf_upsample: D~ is empty at level %d", fine->level);
    return VINP_E_NO_SOURCE;
  }
  if (e > b) {
    k_upsample<<<nblk(e - b, 256), 256, 0, S(stream)>>>(args_of(coarse), cn->e, args_of(fine),
                                                        fn->e, fn->n, prm->seed, b, e);
    count_launch();
  }
  return check_launch("vinp_nnf_upsample");
}

}  // extern "C"

namespace vinp {
vinp_status launch_evaluate(const vinp_level* lv, vinp_nnf* nnf, const vinp_params* prm, int kb,
                            int only_layer, int32_t b, int32_t e, const int32_t* list,
                            unsigned long long* counter, void* stream) {
  vinp_status st = check_nnf_args(lv, "vinp_nnf_evaluate", list ? 0 : b, list ? 0 : e, prm);
  if (st) return st;
  VINP_REQUIRE(nnf && nnf->e && nnf->n, "vinp_nnf_evaluate: null nnf");
  VINP_REQUIRE((kb < 0 && only_layer < 0) || lv->layer, "vinp_nnf_evaluate: layer map required");
  if (e > b) {
    if (kb >= 0)  // K-restricted (onion) launch: warp per target
      k_evaluate_wide<<<nblk((int64_t)(e - b) * 32, VINP_WIDE_BLOCK), VINP_WIDE_BLOCK, 0, S(stream)>>>(
          args_of(lv), nnf->e, nnf->n, nnf->stamp, prm->lambda, kb, only_layer, b, e, list, counter,
          mirror_of(nnf));
    else
      k_evaluate<<<nblk(e - b, VINP_EVAL_BLOCK), VINP_EVAL_BLOCK, 0, S(stream)>>>(
          args_of(lv), nnf->e, nnf->n, nnf->stamp, prm->lambda, kb, only_layer, b, e, list, counter,
          mirror_of(nnf));
    count_launch();
  }
  return check_launch("vinp_nnf_evaluate");
}
// R41 stamps: both buffers or neither; pass in [1, 255]; since in [0, pass)
static vinp_status check_stamps(const vinp_nnf* in, const vinp_nnf* out, int pass, int since,
                                const char* who) {
  VINP_REQUIRE(!in->stamp == !out->stamp, "%s: stamps must be given on both buffers or neither", who);
  VINP_REQUIRE(!in->stamp || in->stamp != out->stamp, "%s: the two buffers share a stamp array", who);
  VINP_REQUIRE(!in->stamp || (pass >= 1 && pass <= 255 && since >= 0 && since < pass),
               "%s: need 1 <= pass <= 255 and 0 <= since < pass (got %d, %d)", who, pass, since);
  return VINP_OK;
}

// smallest level (targets) whose R41-active passes use lv->active; VINP_ACTIVE_MIN in the
// environment overrides the compiled default (the test suite sets 0 to exercise it on small cases)
static int active_min() {
  static const int v = [] {
    const char* s = getenv("VINP_ACTIVE_MIN");
    return s ? atoi(s) : (int)VINP_ACTIVE_MIN;
  }();
  return v;
}

vinp_status launch_propagate(const vinp_level* lv, const vinp_nnf* in, vinp_nnf* out,
                             const vinp_params* prm, int step, int sign, int kb, int only_layer,
                             int32_t b, int32_t e, int pass, int since, const int32_t* list,
                             unsigned long long* counter, void* stream) {
  vinp_status st = check_nnf_args(lv, "vinp_propagate", list ? 0 : b, list ? 0 : e, prm);
  if (st) return st;
  VINP_REQUIRE(in && in->e && out && out->e && in->e != out->e, "vinp_propagate: need two buffers");
  st = check_stamps(in, out, pass, since, "vinp_propagate");
  if (st) return st;
  if (!in->stamp) since = 0;
  VINP_REQUIRE(step >= 1 && sign >= -1 && sign <= 1, "vinp_propagate: bad step/sign");
  VINP_REQUIRE((kb < 0 && only_layer < 0) || lv->layer, "vinp_propagate: layer map required");
  if (e > b) {
    const int pb = e - b >= VINP_PROP_BIG ? VINP_PROP_BLOCK : VINP_PROP_BLOCK_MID;
    if (kb >= 0)  // K-restricted (onion) launch: warp per target
      k_propagate_wide<<<nblk((int64_t)(e - b) * 32, VINP_WIDE_BLOCK), VINP_WIDE_BLOCK, 0, S(stream)>>>(
          args_of(lv), in->e, out->e, in->stamp, out->stamp, prm->lambda, step, sign, kb, only_layer, b, e,
          pass, since, list, counter, mirror_of(out));
    else {
      // R41 active (a previous same-(step, sign) pass exists): the light all-group-path kernel
      const bool light = VINP_PROP_LIGHT && since > 0;
      // lv->active (whole-range single-GPU passes): flag the targets with a non-stale proposal first
      // (levels below VINP_ACTIVE_MIN targets keep the whole-range kernel: three launches instead
      // of one cost more than they save there; c5 level 4, 335 K targets: 16.5 vs 21.1 ms per step)
      uint32_t* active = (light && lv->active && !list && only_layer < 0 && !in->mirror && !out->mirror &&
                          e - b >= active_min())
                             ? lv->active : nullptr;
      if (active) {
        if (cudaMemsetAsync(active, 0, sizeof(uint32_t), S(stream)) != cudaSuccess)
          return check_launch("vinp_propagate(active)");
        const int32_t n = lv->n_targets;
        k_prop_mark<<<nblk(n, 256), 256, 0, S(stream)>>>(args_of(lv), in->e, out->e, in->stamp, out->stamp, active,
                                                         step, sign, since, b, e, n);
        k_prop_compact<<<nblk((int64_t)active_bitmap_words(n), 256), 256, 0, S(stream)>>>(active, n);
        count_launch();
        count_launch();
      }
#define VINP_PROP_LAUNCH(NC, L)                                                                     \
  k_propagate<NC, L><<<nblk(e - b, pb), pb, 0, S(stream)>>>(args_of(lv), in->e, out->e, in->stamp,      \
                                                            out->stamp, prm->lambda, step, sign, kb,     \
                                                            only_layer, b, e, pass, since, list, counter, \
                                                            mirror_of(out), active)
      if (sign == 0) {
        if (light) VINP_PROP_LAUNCH(6, true); else VINP_PROP_LAUNCH(6, false);
      } else {
        if (light) VINP_PROP_LAUNCH(3, true); else VINP_PROP_LAUNCH(3, false);
      }
#undef VINP_PROP_LAUNCH
    }
    count_launch();
  }
  return check_launch("vinp_propagate");
}
}  // namespace vinp

extern "C" {
vinp_status vinp_nnf_evaluate(const vinp_level* lv, vinp_nnf* nnf, const vinp_params* prm, int kb,
                              int only_layer, int32_t b, int32_t e, unsigned long long* counter,
                              void* stream) {
  VINP_NVTX();
  return launch_evaluate(lv, nnf, prm, kb, only_layer, b, e, nullptr, counter, stream);
}

vinp_status vinp_propagate(const vinp_level* lv, const vinp_nnf* in, vinp_nnf* out,
                           const vinp_params* prm, int step, int sign, int kb, int only_layer,
                           int32_t b, int32_t e, int pass, int since, unsigned long long* counter,
                           void* stream) {
  VINP_NVTX();
  return launch_propagate(lv, in, out, prm, step, sign, kb, only_layer, b, e, pass, since, nullptr,
                          counter, stream);
}

}  // extern "C"

namespace vinp {
vinp_status launch_random_search(const vinp_level* lv, const vinp_nnf* in, vinp_nnf* out,
                                 const vinp_params* prm, uint32_t outer_code, int pm_iter, int kb,
                                 int only_layer, int32_t b, int32_t e, int pass, const int32_t* list,
                                 unsigned long long* counter, void* stream) {
  vinp_status st = check_nnf_args(lv, "vinp_random_search", list ? 0 : b, list ? 0 : e, prm);
  if (st) return st;
  VINP_REQUIRE(in && in->e && out && out->e && in->e != out->e, "vinp_random_search: need two buffers");
  st = check_stamps(in, out, pass, 0, "vinp_random_search");
  if (st) return st;
  VINP_REQUIRE(prm->rho > 0 && prm->rho < 1, "vinp_random_search: rho must lie in (0,1)");
  VINP_REQUIRE((kb < 0 && only_layer < 0) || lv->layer, "vinp_random_search: layer map required");
  Radii r = make_radii(lv, prm);
  if (r.M < 0) {
    set_error("vinp_random_search: more than 32 random-search radii R_i = rmax rho^i >= 1 (rho too close to 1)");
    return VINP_E_UNSUPPORTED;
  }
  if (e > b && kb >= 0) {  // K-restricted (onion) launch: warp per target (M <= 32 lanes)
    k_random_search_wide<<<nblk((int64_t)(e - b) * 32, VINP_WIDE_BLOCK), VINP_WIDE_BLOCK, 0, S(stream)>>>(
        args_of(lv), in->e, out->e, in->stamp, out->stamp, prm->lambda, r, prm->seed, outer_code, pm_iter, kb,
        only_layer, b, e, pass, list, counter, mirror_of(out));
    count_launch();
  } else if (e > b) {
    cudaStream_t cs = S(stream);
    LevelArgs la = args_of(lv);
    const bool small = (e - b) < VINP_RS_SMALL;
#define VINP_RS2(NC, WPB, TPW)                                                                       \
  k_random_search<NC, WPB, TPW><<<nblk(e - b, TPW * WPB), 32 * WPB, 0, cs>>>(                           \
      la, in->e, out->e, in->stamp, out->stamp, prm->lambda, r, prm->seed, outer_code, pm_iter, only_layer, b, e, \
      pass, list, counter, mirror_of(out))
#define VINP_RS(NC, WPB)          \
  do {                            \
    if (small)                    \
      VINP_RS2(NC, WPB, 8);       \
    else                          \
      VINP_RS2(NC, WPB, 32);      \
  } while (0)
    if (r.M <= 8)
      VINP_RS(8, VINP_RS_WPB);
    else if (r.M <= 12)
      VINP_RS(12, VINP_RS_WPB);
    else if (r.M <= 16)
      VINP_RS(16, 4);
    else
      VINP_RS(32, 2);
#undef VINP_RS
#undef VINP_RS2
    count_launch();
  }
  return check_launch("vinp_random_search");
}
}  // namespace vinp

extern "C" {
vinp_status vinp_random_search(const vinp_level* lv, const vinp_nnf* in, vinp_nnf* out,
                               const vinp_params* prm, uint32_t outer_code, int pm_iter, int kb,
                               int only_layer, int32_t b, int32_t e, int pass,
                               unsigned long long* counter, void* stream) {
  VINP_NVTX();
  return launch_random_search(lv, in, out, prm, outer_code, pm_iter, kb, only_layer, b, e, pass, nullptr,
                              counter, stream);
}

vinp_status vinp_ann_search(const vinp_level* lv, vinp_nnf* a, vinp_nnf* b, const vinp_params* prm,
                            uint32_t outer_code, int K, const int32_t* steps, int n_steps,
                            int sign_policy, int kb, int only_layer, unsigned long long* counter,
                            void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(sign_policy == 0 || sign_policy == 1, "vinp_ann_search: bad sign_policy");
  VINP_REQUIRE(a && b && steps && n_steps >= 0 && n_steps <= 16 && K >= 0, "vinp_ann_search: bad args");
  vinp_nnf ua = *a, ub = *b;
  if ((int64_t)K * (n_steps + 1) > 255) ua.stamp = ub.stamp = nullptr;  // pass index would overflow u8
  vinp_status st = vinp_nnf_evaluate(lv, &ua, prm, kb, only_layer, 0, lv->n_targets, counter, stream);
  if (st) return st;
  vinp_nnf* cur = &ua;
  vinp_nnf* nxt = &ub;
  PassClock clk;
  for (int k = 1; k <= K; ++k) {
    int sign = sign_policy ? 0 : ((k % 2 == 1) ? 1 : -1);
    for (int i = 0; i < n_steps; ++i) {
      int since = clk.since(steps[i], sign);
      st = vinp_propagate(lv, cur, nxt, prm, steps[i], sign, kb, only_layer, 0, lv->n_targets, clk.pass,
                          since, counter, stream);
      if (st) return st;
      clk.tick(steps[i], sign);
      std::swap(cur, nxt);
    }
    st = vinp_random_search(lv, cur, nxt, prm, outer_code, k, kb, only_layer, 0, lv->n_targets, clk.pass,
                            counter, stream);
    if (st) return st;
    clk.tick(0, 2);
    std::swap(cur, nxt);
  }
  cur = cur == &ua ? a : b;
  if (cur != a && lv->n_targets > 0) {
    if (cudaMemcpyAsync(a->e, cur->e, sizeof(uint64_t) * lv->n_targets, cudaMemcpyDeviceToDevice,
                        S(stream)) != cudaSuccess)
      return check_launch("vinp_ann_search(copy)");
  }
  return VINP_OK;
}

size_t vinp_brute_force_ws_bytes(const vinp_level* lv) {
  (void)lv;
  return 0;  // the CUDA-core form needs no workspace
}

vinp_status vinp_brute_force(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm, int32_t b,
                             int32_t e, void* ws, size_t ws_bytes, void* stream) {
  VINP_NVTX();
  vinp_status st = check_nnf_args(lv, "vinp_brute_force", b, e, prm);
  if (st) return st;
  VINP_REQUIRE(out && out->e && out->n, "vinp_brute_force: null nnf");
  (void)ws;
  (void)ws_bytes;
  if (lv->n_sources <= 0) {
    set_error("vinp_brute_force: D~ is empty");
    return VINP_E_NO_SOURCE;
  }
  if (e > b) {
    k_brute_force<<<e - b, 32 * kWarpsPerBlock, 0, S(stream)>>>(args_of(lv), out->e, out->n,
                                                                 prm->lambda, b, e, nullptr);
    count_launch();
  }
  return check_launch("vinp_brute_force");
}

vinp_status vinp_brute_force_list(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm,
                                  const int32_t* list, int32_t n, void* stream) {
  VINP_NVTX();
  vinp_status st = check_nnf_args(lv, "vinp_brute_force_list", 0, 0, prm);
  if (st) return st;
  VINP_REQUIRE(out && out->e && out->n, "vinp_brute_force_list: null nnf");
  VINP_REQUIRE(n >= 0 && (n == 0 || list), "vinp_brute_force_list: null list or negative count");
  VINP_REQUIRE(n <= lv->n_targets, "vinp_brute_force_list: more list entries than targets");
  if (lv->n_sources <= 0) {
    set_error("vinp_brute_force_list: D~ is empty");
    return VINP_E_NO_SOURCE;
  }
  if (n > 0) {
    k_brute_force<<<n, 32 * kWarpsPerBlock, 0, S(stream)>>>(args_of(lv), out->e, out->n, prm->lambda, 0,
                                                             n, list);
    count_launch();
  }
  return check_launch("vinp_brute_force_list");
}

size_t vinp_active_ws_bytes(const vinp_level* lv) {
  if (!lv || lv->n_targets < 0) return 0;
  return 4 * (8 + active_bitmap_words(lv->n_targets) + (size_t)lv->n_targets);
}

vinp_status vinp_patch_sums(const vinp_level* lv, int which, int32_t b, int32_t e, void* stream) {
  VINP_NVTX();
  vinp_status st = check_level(lv, "vinp_patch_sums");
  if (st) return st;
  VINP_REQUIRE(lv->psum, "vinp_patch_sums: lv->psum is NULL");
  VINP_REQUIRE(which == 0 || which == 1, "vinp_patch_sums: which must be 0 (all voxels) or 1 (targets)");
  if (which == 0) {
    k_patch_sums_dense<<<nblk(lv->W * lv->H, 128), 128, 0, S(stream)>>>(args_of(lv),
                                                                        reinterpret_cast<uint4*>(lv->psum));
    count_launch();
  } else {
    VINP_REQUIRE(lv->targets && b >= 0 && b <= e && e <= lv->n_targets, "vinp_patch_sums: bad slot range");
    if (e > b) {
      k_patch_sums_targets<<<nblk(e - b, 128), 128, 0, S(stream)>>>(args_of(lv), reinterpret_cast<uint4*>(lv->psum),
                                                                    b, e);
      count_launch();
    }
  }
  return check_launch("vinp_patch_sums");
}

vinp_status vinp_patch_ssd(const vinp_level* lv, const int32_t* p, const int32_t* q, int64_t n,
                           const vinp_params* prm, int kb, uint32_t* D, uint8_t* cnt, void* stream) {
  VINP_NVTX();
  vinp_status st = check_level(lv, "vinp_patch_ssd");
  if (st) return st;
  VINP_REQUIRE(p && q && D && cnt && prm && n >= 0, "vinp_patch_ssd: bad args");
  VINP_REQUIRE(kb < 0 || lv->layer, "vinp_patch_ssd: layer map required");
  if (n > 0) {
    k_patch_ssd<<<nblk(n, kWarpsPerBlock), 32 * kWarpsPerBlock, 0, S(stream)>>>(
        args_of(lv), p, q, n, prm->lambda, kb, D, cnt);
    count_launch();
  }
  return check_launch("vinp_patch_ssd");
}

vinp_status vinp_philox(const uint32_t* ctr, int64_t n, uint64_t seed, uint32_t* out, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(ctr && out && n >= 0, "vinp_philox: bad args");
  if (n > 0) {
    k_philox<<<nblk(n, 256), 256, 0, S(stream)>>>((const uint4*)ctr, n, seed, (uint4*)out);
    count_launch();
  }
  return check_launch("vinp_philox");
}

}  // extern "C"
