// bf_tc.cu — exact brute-force NN on the 5th-generation tensor cores (row a13, optional mode).
//
// For full patches (N_p inside Omega, K = Omega) the integer distance of Eq. 9 (R24) splits as
//   D(p,q) = E(p) + E(q) - 2 [ 4 X_c(p,q) + lambda X_t(p,q) ],
//   E(x)   = 4 sum ||u||^2 + lambda sum ||T_q||^2 over the patch,   X = patch dot products,
// so argmin_q D(p,q) over q in D~ is an integer GEMM of u8 patch vectors (implicit im2col):
// colour K = 125*3 -> 384, texture K = 125*2 -> 256, two s32 accumulators in TMEM, combined
// exactly in the epilogue with E(q), running (D, index) minimum per target row (ties -> smallest
// index, as the oracle's exhaustive scan).  tcgen05.mma.cta_group::1.kind::i8, M = 128 targets,
// N = 128 sources per MMA, operands staged K-major (no swizzle) in shared memory.
#include <vector>

#include "common.cuh"
#include "tc.cuh"

namespace vinp {

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// ------------------------------------------------------------------ probe: C = A B^T (u8 -> s32)
// A [128][K], B [128][K] row-major (K-major), K % 32 == 0, K <= 512.
__global__ void __launch_bounds__(128) k_tc_gemm_probe(const uint8_t* __restrict__ A,
                                                       const uint8_t* __restrict__ B, int K,
                                                       int32_t* __restrict__ C) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;
  uint8_t* sB = sm + 128 * K;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int nch = K / 16;
  for (int c = tid; c < 128 * nch; c += 128) {
    int m = c / nch, kc = c % nch;
    int off = (m >> 3) * 128 + kc * (128 * 16) + (m & 7) * 16;
    tc::cp16(sA + off, A + (size_t)m * K + kc * 16);
    tc::cp16(sB + off, B + (size_t)m * K + kc * 16);
  }
  tc::cp_wait_all();
  tc::fence_proxy_async();
  if (warp == 0) tc::tmem_alloc(&tmem_base, 128);
  if (tid == 0) tc::mbar_init(&mbar, 1);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  uint32_t tm = tmem_base;
  if (tid == 0) {
    uint32_t id = tc::idesc_u8(128, 128);
    uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB);
    for (int j = 0; j < K / 32; ++j) {
      uint64_t da = tc::desc_kmajor(a0 + 2 * j * 2048, 2048, 128);
      uint64_t db = tc::desc_kmajor(b0 + 2 * j * 2048, 2048, 128);
      tc::mma_u8(tm, da, db, id, j > 0);
    }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tc::tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + 32 * c, v);
    int row = 32 * warp + lane;
#pragma unroll
    for (int j = 0; j < 32; ++j) C[row * 128 + 32 * c + j] = (int32_t)v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tm, 128);
}

// ------------------------------------------------------------------ exact NN on tensor cores
constexpr int kRow = 640;       // bytes per patch row: colour 384 (125*3 + 9 pad), texture 256 (250 + 6)
constexpr int kColK = 384, kTexK = 256;
constexpr int kTile = 128;      // M (targets) and N (sources) per tile
// Energies and distances fit in int32: D <= 4*125*3*255^2 + 126*125*2*255^2 = 2,145,825,000 < 2^31
// for lambda <= 126 (vinp.h), hence also E(q) - 2X = D - E(p).  Padded rows get 2^31 - 1, which
// no real E(q) - 2X reaches, so they never win (X = 0 for their zero operands).
constexpr int32_t kEPad = 0x7fffffff;

__device__ __forceinline__ bool full_patch(const Geo& g, int x, int y, int t) {
  return x >= 2 && x < g.W - 2 && y >= 2 && y < g.H - 2 && t >= 2 && t < g.T - 2;
}

// im2col of the patch around voxel p (a full patch) in the TILED core-matrix layout of tc.cuh: rows are
// grouped in tiles of TR rows; a tile is [colour: 24 K-chunks x TR/8 core matrices][texture: 16 x
// TR/8], K byte k of row r at  part + (k/16)*TR*16 + (r/8)*128 + (r%8)*16 + k%16, so that a whole tile
// is one contiguous block that a bulk (TMA) copy lands in shared memory ready for tcgen05.mma.
// energy[i] = 4 sum c^2 + lambda sum t^2 (int32, see kEPad; padded rows: zeros, energy kEPad).
__device__ __forceinline__ size_t tiled_off(int i, int k, int TR) {
  int tile = i / TR, r = i % TR;
  size_t base = (size_t)tile * TR * kRow;
  if (k >= kColK) {
    base += (size_t)TR * kColK;
    k -= kColK;
  }
  return base + (size_t)(k >> 4) * TR * 16 + (r >> 3) * 128 + (r & 7) * 16 + (k & 15);
}

__global__ void k_im2col_tiled(const uint64_t* __restrict__ vox, Geo g, const int32_t* __restrict__ pos,
                               const int32_t* __restrict__ idx, int32_t n, int32_t npad, int lambda, int TR,
                               uint8_t* __restrict__ rows, int32_t* __restrict__ energy) {
  int i = blockIdx.x;  // one block (128 threads) per row
  if (i >= npad) return;
  if (i >= n) {
    for (int k = threadIdx.x; k < kRow; k += blockDim.x) rows[tiled_off(i, k, TR)] = 0;
    if (threadIdx.x == 0) energy[i] = kEPad;
    return;
  }
  int p = pos[idx ? idx[i] : i];
  int px, py, pt;
  decode(g, p, px, py, pt);
  uint32_t ec = 0, et = 0;
  int v = threadIdx.x;
  if (v < kPatch) {
    int dx, dy, dt;
    voff(v, dx, dy, dt);
    // voxels of a clipped (border) patch outside Omega are zero rows of the contraction
    uint64_t w = inside(g, px + dx, py + dy, pt + dt) ? vox[p + dt * g.HW + dy * g.W + dx] : 0ull;
    uint32_t c0 = w & 255, c1 = (w >> 8) & 255, c2 = (w >> 16) & 255, t0 = (w >> 32) & 255, t1 = (w >> 40) & 255;
    rows[tiled_off(i, 3 * v, TR)] = (uint8_t)c0;
    rows[tiled_off(i, 3 * v + 1, TR)] = (uint8_t)c1;
    rows[tiled_off(i, 3 * v + 2, TR)] = (uint8_t)c2;
    rows[tiled_off(i, kColK + 2 * v, TR)] = (uint8_t)t0;
    rows[tiled_off(i, kColK + 2 * v + 1, TR)] = (uint8_t)t1;
    ec = c0 * c0 + c1 * c1 + c2 * c2;
    et = t0 * t0 + t1 * t1;
  }
  for (int k = 375 + threadIdx.x; k < kColK; k += blockDim.x) rows[tiled_off(i, k, TR)] = 0;
  for (int k = kColK + 250 + threadIdx.x; k < kRow; k += blockDim.x) rows[tiled_off(i, k, TR)] = 0;
  ec = __reduce_add_sync(kFull, ec);
  et = __reduce_add_sync(kFull, et);
  __shared__ uint32_t sc[4], st[4];
  if ((threadIdx.x & 31) == 0) { sc[threadIdx.x >> 5] = ec; st[threadIdx.x >> 5] = et; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t c = 0, t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { c += sc[w]; t += st[w]; }
    energy[i] = (int32_t)(4 * c + (uint64_t)lambda * t);
  }
}

// Warp-specialised exact-NN GEMM.  CTA = (m tile of 128 targets, chunk of source tiles of 64).
// warp 0: producer — bulk (TMA) copies of the A tile (once) and of B tiles into a 2-stage ring;
// warp 1: MMA issuer — 12 colour + 8 texture tcgen05.mma kind::i8 (M=128, N=64, K=32) per B tile
//         into a 2-stage TMEM accumulator ring (stage s: colour cols s*128+[0,64), texture +64);
// warps 2-5: epilogue — tcgen05.ld of their 32 TMEM lanes, D = E(q) - 2(4 X_c + lambda X_t), running
//         (D, index) minimum per target row (strict <, ascending sources: first minimum).
// Barriers: a_full; b_full[2] / b_empty[2] (producer <-> MMA); acc_full[2] / acc_empty[2] (MMA <->
// epilogue, 128 arrivals).  All waits are bounded (trap instead of hang).
constexpr int kTA = 128, kTB = 128;
constexpr int kEpiWarps = 8, kBfThreads = 64 + 32 * kEpiWarps;  // producer, MMA, 8 epilogue warps
constexpr uint32_t kABytes = kTA * kRow, kBBytes = kTB * kRow;
constexpr uint32_t kBColBytes = kTB * kColK, kBTexBytes = kTB * kTexK;  // the two parts of a B tile

// N = 128 source columns per MMA (M128 N128 K32: half the A re-reads from shared memory per MAC
// of N = 64).  A source tile (80 KB) is streamed in its two parts — colour (48 KB) into shared
// stage 0, texture (32 KB) into stage 1 — so the next tile's colour part loads while this tile's
// texture MMAs run: 80 KB (A) + 2 x 48 KB of shared memory.  TMEM: 2 accumulator stages x (128
// colour + 128 texture columns) = 512 columns.
__global__ void __launch_bounds__(kBfThreads, 1) k_bf_tc2(const uint8_t* __restrict__ A, const int32_t* __restrict__ Ep,
                                                          const uint8_t* __restrict__ B, const int32_t* __restrict__ Eq,
                                                          int nb_tiles, int tiles_per_chunk, int lambda, int32_t mpad,
                                                          int32_t nsrc, uint64_t* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;
  uint8_t* sB[2] = {sm + kABytes, sm + kABytes + kBColBytes};  // colour part, texture part
  // barriers: a_full; b_full[2] / b_empty[2] (colour / texture part); acc_full[2] / acc_empty[2]
  __shared__ uint64_t bar[9];
  uint64_t* const bfull = bar + 1;
  uint64_t* const bempty = bar + 3;
  uint64_t* const afull = bar + 5;
  uint64_t* const aempty = bar + 7;
  __shared__ uint32_t tmem_base;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int mt = blockIdx.x;
  int t0 = blockIdx.y * tiles_per_chunk, t1 = min(nb_tiles, t0 + tiles_per_chunk);
  int nt = max(0, t1 - t0);
  if (tid == 0) {
    for (int k = 0; k < 7; ++k) tc::mbar_init(&bar[k], 1);
    for (int k = 0; k < 2; ++k) tc::mbar_init(&aempty[k], 32 * kEpiWarps);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tmem_base;
  if (warp == 0) {
    if (lane == 0) {
      const uint8_t* ga = A + (size_t)mt * kABytes;
      tc::mbar_expect_tx(&bar[0], kABytes);
      for (uint32_t o = 0; o < kABytes; o += 16384) tc::bulk_g2s(sA + o, ga + o, min(16384u, kABytes - o), &bar[0]);
      for (int i = 0; i < nt; ++i) {
        const uint8_t* gb = B + (size_t)(t0 + i) * kBBytes;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          const uint32_t nb = part ? kBTexBytes : kBColBytes;
          const uint8_t* src = gb + (part ? kBColBytes : 0);
          tc::mbar_wait(&bempty[part], (i & 1) ^ 1);
          tc::mbar_expect_tx(&bfull[part], nb);
          for (uint32_t o = 0; o < nb; o += 16384) tc::bulk_g2s(sB[part] + o, src + o, min(16384u, nb - o), &bfull[part]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id = tc::idesc_u8(kTA, kTB);
      const uint32_t ac = tc::smem_u32(sA), at = ac + kTA * kColK;
      const uint32_t bc = tc::smem_u32(sB[0]), bt = tc::smem_u32(sB[1]);
      tc::mbar_wait(&bar[0], 0);
      for (int i = 0; i < nt; ++i) {
        const int sa = i & 1;
        const uint32_t dc = tm + sa * 256, dt = dc + 128;
        tc::mbar_wait(&aempty[sa], ((i >> 1) & 1) ^ 1);
        tc::mbar_wait(&bfull[0], i & 1);
        tc::fence_after();
#pragma unroll
        for (int j = 0; j < kColK / 32; ++j)
          tc::mma_u8(dc, tc::desc_kmajor(ac + 2 * j * (kTA * 16), kTA * 16, 128),
                     tc::desc_kmajor(bc + 2 * j * (kTB * 16), kTB * 16, 128), id, j > 0);
        tc::commit(&bempty[0]);  // colour part free once these MMAs have read it
        tc::mbar_wait(&bfull[1], i & 1);
        tc::fence_after();
#pragma unroll
        for (int j = 0; j < kTexK / 32; ++j)
          tc::mma_u8(dt, tc::desc_kmajor(at + 2 * j * (kTA * 16), kTA * 16, 128),
                     tc::desc_kmajor(bt + 2 * j * (kTB * 16), kTB * 16, 128), id, j > 0);
        tc::commit(&bempty[1]);  // texture part free
        tc::commit(&afull[sa]);  // accumulator stage ready
      }
    }
  } else {
    // 8 epilogue warps: warp w reads TMEM lane quarter w % 4 (the hardware rule); the two warps of
    // a quarter take 64 of the tile's 128 columns each, in two chunks of 32.  Per row the minimum
    // over sources of s = E(q) - 2 (4 X_c + lambda X_t) = D - E(p) (int32, exact: D < 2^31 for
    // lambda <= 126), first index on ties; per chunk one min per column, and the first-index search
    // only when the chunk improves the running minimum (strict, so earlier columns win ties).
    const int q = warp & 3;
    const int h = warp >= 2 + kEpiWarps / 2 ? 1 : 0;
    const int row = 32 * q + lane;
    int32_t bestS = 0x7fffffff;
    int bestI = 0x7fffffff;
    const uint32_t lam2 = 2u * (uint32_t)lambda;
    for (int i = 0; i < nt; ++i) {
      const int sa = i & 1;
      tc::mbar_wait(&afull[sa], (i >> 1) & 1);
      tc::fence_after();
#pragma unroll 1
      for (int ch = 0; ch < 2; ++ch) {
        const int col = 64 * h + 32 * ch;
        uint32_t c[32], x[32];
        uint32_t base = tm + ((uint32_t)(32 * q) << 16) + sa * 256 + col;
        tc::tmem_ld32x2(base, base + 128, c, x);
        const int cbase = (t0 + i) * kTB + col;
        const int4* E4 = reinterpret_cast<const int4*>(Eq + cbase);  // 16-B aligned: cbase % 4 == 0
        int32_t sv[32];
        int32_t tmin = 0x7fffffff;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          int4 ev = __ldg(E4 + j4);
          const int32_t e4[4] = {ev.x, ev.y, ev.z, ev.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 4 * j4 + u;
            sv[j] = (int32_t)((uint32_t)e4[u] - lam2 * x[j] - 8u * c[j]);  // exact mod 2^32 (2 IMADs)
            tmin = min(tmin, sv[j]);
          }
        }
        if (tmin < bestS) {
          int jf = 31;
#pragma unroll
          for (int j = 31; j >= 0; --j)
            if (sv[j] == tmin) jf = j;
          bestS = tmin;
          bestI = cbase + jf;
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&aempty[sa]);  // accumulator stage drained (by this thread)
    }
    uint32_t bestD = (uint32_t)Ep[(size_t)mt * kTA + row] + (uint32_t)bestS;  // = D, exact mod 2^32
    // merge the two column halves of each row: lexicographic (D, index) minimum
    __shared__ uint32_t mD[kTA];
    __shared__ int mI[kTA];
    if (h == 1) {
      mD[row] = bestD;
      mI[row] = bestI;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiWarps));  // epilogue warps only
    if (h == 0) {
      uint32_t D2 = mD[row];
      int I2 = mI[row];
      // (a half that saw only padding columns has no index: skip it)
      if (I2 != 0x7fffffff && (bestI == 0x7fffffff || D2 < bestD || (D2 == bestD && I2 < bestI))) {
        bestD = D2;
        bestI = I2;
      }
      uint64_t packed = bestI == 0x7fffffff ? ~0ull : (((uint64_t)bestD << 32) | (uint32_t)bestI);
      out[(size_t)blockIdx.y * mpad + (size_t)mt * kTA + row] = packed;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_free(tm, 512);
}

// Clip pattern of a target patch: how many voxel layers fall outside Omega on each side of each
// axis (0..2 each); pid = xl + 3xh + 9yl + 27yh + 81tl + 243th, 0 = full patch.
__device__ __forceinline__ int clip_pid(const Geo& g, int x, int y, int t) {
  int xl = max(0, 2 - x), xh = max(0, x + 3 - g.W), yl = max(0, 2 - y), yh = max(0, y + 3 - g.H);
  int tl = max(0, 2 - t), th = max(0, t + 3 - g.T);
  return xl + 3 * xh + 9 * yl + 27 * yh + 81 * tl + 243 * th;
}
constexpr int kPids = 729;

__global__ void k_pid_count(const int32_t* __restrict__ targets, Geo g, int32_t b, int32_t e,
                            int32_t* __restrict__ cnt) {
  int i = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e) return;
  int x, y, t;
  decode(g, targets[i], x, y, t);
  atomicAdd(cnt + clip_pid(g, x, y, t), 1);
}
// slots grouped by pattern (order within a group is irrelevant: targets are independent)
__global__ void k_pid_scatter(const int32_t* __restrict__ targets, Geo g, int32_t b, int32_t e,
                              int32_t* __restrict__ cursor, int32_t* __restrict__ list) {
  int i = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e) return;
  int x, y, t;
  decode(g, targets[i], x, y, t);
  list[atomicAdd(cursor + clip_pid(g, x, y, t), 1)] = i;
}
// per-source energy over the sub-box of a clip pattern: 4 sum c^2 + lambda sum t^2
__global__ void k_energy_box(const uint64_t* __restrict__ vox, Geo g, const int32_t* __restrict__ sources,
                             int32_t n, int32_t npad, int lambda, int pid, int32_t* __restrict__ E) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npad) return;
  if (i >= n) { E[i] = kEPad; return; }
  int xl = pid % 3, xh = pid / 3 % 3, yl = pid / 9 % 3, yh = pid / 27 % 3, tl = pid / 81 % 3, th = pid / 243;
  int q = sources[i];
  uint64_t c = 0, tt = 0;
  for (int dt = -2 + tl; dt <= 2 - th; ++dt)
    for (int dy = -2 + yl; dy <= 2 - yh; ++dy)
      for (int dx = -2 + xl; dx <= 2 - xh; ++dx) {
        uint64_t w = vox[q + dt * g.HW + dy * g.W + dx];
        uint32_t c0 = w & 255, c1 = (w >> 8) & 255, c2 = (w >> 16) & 255, t0 = (w >> 32) & 255, t1 = (w >> 40) & 255;
        c += c0 * c0 + c1 * c1 + c2 * c2;
        tt += t0 * t0 + t1 * t1;
      }
  E[i] = (int32_t)(4 * c + (uint64_t)lambda * tt);
}

// merge the split minima (lexicographic (D, index) = smallest D, then smallest source index)
__global__ void k_bf_merge(const uint64_t* __restrict__ part, int splits, int32_t mpad, int32_t m,
                           const int32_t* __restrict__ list, const int32_t* __restrict__ sources,
                           uint64_t* __restrict__ ee, uint8_t* __restrict__ en, int nvox) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint64_t best = ~0ull;
  for (int s = 0; s < splits; ++s) best = min(best, part[(size_t)s * mpad + i]);
  int slot = list[i];
  ee[slot] = pack_e((uint32_t)(best >> 32), sources[(uint32_t)best]);
  en[slot] = (uint8_t)nvox;
}

}  // namespace vinp

using namespace vinp;

extern "C" {

size_t vinp_brute_force_tc_ws_bytes(const vinp_level* lv, int32_t b, int32_t e) {
  if (!lv) return 0;
  int64_t m = std::max<int64_t>(0, e - b), mpad = (m + kTile - 1) / kTile * kTile;
  int64_t npad = ((int64_t)lv->n_sources + kTile - 1) / kTile * kTile;
  int64_t splits = (npad / 64) / ((64ll << 20) / (64 * kRow)) + 2;  // >= the number of 64 MB source chunks
  return (size_t)((mpad + 128 * 8) * kRow + (mpad + 128 * 8) * 8 + npad * kRow + 2 * npad * 8 + mpad * 4 +
                  2 * 729 * 4 + 64 + splits * (mpad + 128 * 8) * 8 + 4096);
}

// implemented in ann.cu: CUDA-core exact NN over an explicit slot list
vinp_status vinp_brute_force_list(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm,
                                  const int32_t* list, int32_t n, void* stream);

vinp_status vinp_brute_force_tc(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm, int32_t b,
                                int32_t e, void* ws, size_t ws_bytes, void* stream) {
  VINP_NVTX();
  vinp_status st = check_level(lv, "vinp_brute_force_tc");
  if (st) return st;
  VINP_REQUIRE(out && out->e && out->n && prm && ws && lv->targets && lv->sources, "vinp_brute_force_tc: bad args");
  VINP_REQUIRE(b >= 0 && e <= lv->n_targets && b <= e, "vinp_brute_force_tc: bad slot range");
  VINP_REQUIRE(prm->lambda >= 0 && prm->lambda <= 126, "vinp_brute_force_tc: lambda outside [0,126]");
  VINP_REQUIRE(ws_bytes >= vinp_brute_force_tc_ws_bytes(lv, b, e), "vinp_brute_force_tc: ws too small");
  if (lv->n_sources <= 0) {
    set_error("vinp_brute_force_tc: D~ is empty");
    return VINP_E_NO_SOURCE;
  }
  if (e == b) return VINP_OK;
  cudaStream_t s = S(stream);
  Geo g = geo_of(lv);
  int64_t m_all = e - b, mpad = (m_all + kTile - 1) / kTile * kTile;
  int64_t npad = ((int64_t)lv->n_sources + kTile - 1) / kTile * kTile;
  int64_t np = ((int64_t)lv->n_sources + kTB - 1) / kTB * kTB;
  char* w = (char*)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
  uint8_t* A = (uint8_t*)w; w += (mpad + kTA * 8) * kRow;
  uint8_t* B = (uint8_t*)w; w += npad * kRow;
  int32_t* Ep = (int32_t*)w; w += (mpad + kTA * 8) * 8;
  int32_t* Eq = (int32_t*)w; w += npad * 8;
  int32_t* Eb = (int32_t*)w; w += npad * 8;  // per-pattern source energies
  int32_t* list = (int32_t*)w; w += mpad * 4;
  int32_t* cnt = (int32_t*)(((uintptr_t)w + 63) & ~(uintptr_t)63); w = (char*)(cnt + 2 * kPids);
  uint64_t* part = (uint64_t*)(((uintptr_t)w + 63) & ~(uintptr_t)63);
  // 1. group the targets of [b, e) by clip pattern (one sync for the group sizes)
  cudaMemsetAsync(cnt, 0, sizeof(int32_t) * 2 * kPids, s);
  k_pid_count<<<nblk(m_all, 256), 256, 0, s>>>(lv->targets, g, b, e, cnt);
  std::vector<int32_t> hc(kPids);
  if (cudaMemcpyAsync(hc.data(), cnt, sizeof(int32_t) * kPids, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return check_launch("vinp_brute_force_tc(count)");
  std::vector<int32_t> off(kPids + 1, 0);
  for (int k = 0; k < kPids; ++k) off[k + 1] = off[k] + hc[k];
  cudaMemcpyAsync(cnt + kPids, off.data(), sizeof(int32_t) * kPids, cudaMemcpyHostToDevice, s);
  k_pid_scatter<<<nblk(m_all, 256), 256, 0, s>>>(lv->targets, g, b, e, cnt + kPids, list);
  count_launch(2);
  // 2. source im2col (tiles of 64) once, with the full-patch energies
  k_im2col_tiled<<<(int)np, 128, 0, s>>>(lv->vox, g, lv->sources, nullptr, lv->n_sources, (int)np, prm->lambda,
                                         kTB, B, Eq);
  count_launch();
  int nb_tiles = (int)(np / kTB);
  int per = std::max(1, std::min(nb_tiles, (int)((64ll << 20) / kBBytes)));
  int chunks = (nb_tiles + per - 1) / per;
  size_t smem = kABytes + 2 * (size_t)kBColBytes;
  cudaFuncSetAttribute(k_bf_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // 3. one warp-specialised tensor-core GEMM + exact argmin per clip pattern
  for (int pid = 0; pid < kPids; ++pid) {
    int32_t m = hc[pid];
    if (m == 0) continue;
    int32_t mp = (m + kTA - 1) / kTA * kTA;
    const int32_t* lst = list + off[pid];
    const int32_t* E = Eq;
    if (pid != 0) {
      k_energy_box<<<nblk(np, 256), 256, 0, s>>>(lv->vox, g, lv->sources, lv->n_sources, (int)np, prm->lambda, pid, Eb);
      count_launch();
      E = Eb;
    }
    int nvox = (5 - pid % 3 - pid / 3 % 3) * (5 - pid / 9 % 3 - pid / 27 % 3) * (5 - pid / 81 % 3 - pid / 243);
    k_im2col_tiled<<<mp, 128, 0, s>>>(lv->vox, g, lv->targets, lst, m, mp, prm->lambda, kTA, A, Ep);
    k_bf_tc2<<<dim3(mp / kTA, chunks), kBfThreads, smem, s>>>(A, Ep, B, E, nb_tiles, per, prm->lambda, mp,
                                                           lv->n_sources, part);
    k_bf_merge<<<nblk(m, 256), 256, 0, s>>>(part, chunks, mp, m, lst, lv->sources, out->e, out->n, nvox);
    count_launch(3);
  }
  return check_launch("vinp_brute_force_tc");
}

vinp_status vinp_tc_gemm_u8(const uint8_t* A, const uint8_t* B, int K, int32_t* C, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(A && B && C && K > 0 && K % 32 == 0 && K <= 512, "vinp_tc_gemm_u8: bad arguments");
  size_t smem = 2 * 128 * (size_t)K;
  cudaFuncSetAttribute(k_tc_gemm_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tc_gemm_probe<<<1, 128, smem, S(stream)>>>(A, B, K, C);
  count_launch();
  return check_launch("vinp_tc_gemm_u8");
}

}  // extern "C"
