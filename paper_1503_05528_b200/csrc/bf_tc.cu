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
constexpr int64_t kEPad = 1ll << 40;  // energy of padded source rows: never the minimum

__device__ __forceinline__ bool full_patch(const Geo& g, int x, int y, int t) {
  return x >= 2 && x < g.W - 2 && y >= 2 && y < g.H - 2 && t >= 2 && t < g.T - 2;
}

// im2col row of the patch around voxel p (must be a full patch) + its energy E = 4 sum c^2 + lambda sum t^2
__global__ void k_im2col(const uint64_t* __restrict__ vox, Geo g, const int32_t* __restrict__ pos,
                         const int32_t* __restrict__ idx, int32_t n, int32_t npad, int lambda,
                         uint8_t* __restrict__ rows, int64_t* __restrict__ energy) {
  int i = blockIdx.x;  // one block (128 threads) per row
  if (i >= npad) return;
  uint8_t* row = rows + (size_t)i * kRow;
  if (i >= n) {
    for (int k = threadIdx.x; k < kRow; k += blockDim.x) row[k] = 0;
    if (threadIdx.x == 0) energy[i] = kEPad;
    return;
  }
  int p = pos[idx ? idx[i] : i];
  uint32_t ec = 0, et = 0;
  for (int v = threadIdx.x; v < 128; v += blockDim.x) {
    uint64_t w = 0;
    if (v < kPatch) {
      int dx, dy, dt;
      voff(v, dx, dy, dt);
      w = vox[p + dt * g.HW + dy * g.W + dx];
      uint32_t r = w & 255, gg = (w >> 8) & 255, b = (w >> 16) & 255, tx = (w >> 32) & 255, ty = (w >> 40) & 255;
      row[3 * v] = (uint8_t)r;
      row[3 * v + 1] = (uint8_t)gg;
      row[3 * v + 2] = (uint8_t)b;
      row[kColK + 2 * v] = (uint8_t)tx;
      row[kColK + 2 * v + 1] = (uint8_t)ty;
      ec += r * r + gg * gg + b * b;
      et += tx * tx + ty * ty;
    }
  }
  for (int k = 375 + threadIdx.x; k < kColK; k += blockDim.x) row[k] = 0;
  for (int k = kColK + 250 + threadIdx.x; k < kRow; k += blockDim.x) row[k] = 0;
  ec = __reduce_add_sync(kFull, ec);
  et = __reduce_add_sync(kFull, et);
  __shared__ uint32_t sc[4], st[4];
  if ((threadIdx.x & 31) == 0) { sc[threadIdx.x >> 5] = ec; st[threadIdx.x >> 5] = et; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t c = 0, t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { c += sc[w]; t += st[w]; }
    energy[i] = (int64_t)(4 * c + (uint64_t)lambda * t);
  }
}

// stage a [128][640] row block into shared memory in the core-matrix layout of tc.cuh, separately
// for the colour (K = 384) and texture (K = 256) parts
__device__ __forceinline__ void stage_rows(uint8_t* sc, uint8_t* st, const uint8_t* __restrict__ g) {
  for (int c = threadIdx.x; c < kTile * (kRow / 16); c += blockDim.x) {
    int m = c / (kRow / 16), kc = c % (kRow / 16);
    const uint8_t* src = g + (size_t)m * kRow + kc * 16;
    if (kc < kColK / 16)
      tc::cp16(sc + (m >> 3) * 128 + kc * (kTile * 16) + (m & 7) * 16, src);
    else
      tc::cp16(st + (m >> 3) * 128 + (kc - kColK / 16) * (kTile * 16) + (m & 7) * 16, src);
  }
}

// grid (m tiles, n splits); 128 threads; out[split][row] = (D_partial << 32 | source index) min
__global__ void __launch_bounds__(128, 1) k_bf_tc(const uint8_t* __restrict__ A, const int64_t* __restrict__ Ep,
                                                  const uint8_t* __restrict__ B, const int64_t* __restrict__ Eq,
                                                  int n_tiles, int tiles_per_split, int lambda,
                                                  int32_t mpad, uint64_t* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sAc = sm;
  uint8_t* sAt = sAc + kTile * kColK;
  uint8_t* sBc = sAt + kTile * kTexK;
  uint8_t* sBt = sBc + kTile * kColK;
  int64_t* sE = reinterpret_cast<int64_t*>(sBt + kTile * kTexK);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int mt = blockIdx.x;
  int t0 = blockIdx.y * tiles_per_split, t1 = min(n_tiles, t0 + tiles_per_split);
  stage_rows(sAc, sAt, A + (size_t)mt * kTile * kRow);
  if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
  if (tid == 0) tc::mbar_init(&mbar, 1);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tmem_base;
  const uint32_t id = tc::idesc_u8(kTile, kTile);
  const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
  int64_t best = INT64_MAX;  // (partial D << 32 | index) packed later
  int64_t bestD = INT64_MAX;
  int bestI = 0x7fffffff;
  uint32_t phase = 0;
  for (int nt = t0; nt < t1; ++nt) {
    stage_rows(sBc, sBt, B + (size_t)nt * kTile * kRow);
    sE[tid] = Eq[(size_t)nt * kTile + tid];
    tc::cp_wait_all();
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      uint32_t ac = tc::smem_u32(sAc), at = tc::smem_u32(sAt), bc = tc::smem_u32(sBc), bt = tc::smem_u32(sBt);
#pragma unroll
      for (int j = 0; j < kColK / 32; ++j)
        tc::mma_u8(tm, tc::desc_kmajor(ac + 2 * j * 2048, 2048, 128), tc::desc_kmajor(bc + 2 * j * 2048, 2048, 128),
                   id, j > 0);
#pragma unroll
      for (int j = 0; j < kTexK / 32; ++j)
        tc::mma_u8(tm + kTile, tc::desc_kmajor(at + 2 * j * 2048, 2048, 128),
                   tc::desc_kmajor(bt + 2 * j * 2048, 2048, 128), id, j > 0);
      tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, phase);
    phase ^= 1;
    tc::fence_after();
#pragma unroll 1
    for (int c = 0; c < kTile / 32; ++c) {
      uint32_t vc[32], vt[32];
      tc::tmem_ld32(tm + lane_off + 32 * c, vc);
      tc::tmem_ld32(tm + lane_off + kTile + 32 * c, vt);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        int col = 32 * c + j;
        int64_t d = sE[col] - 2 * (4 * (int64_t)vc[j] + (int64_t)lambda * (int64_t)vt[j]);
        if (d < bestD) {
          bestD = d;
          bestI = nt * kTile + col;
        }
      }
    }
    tc::fence_before();
    __syncthreads();  // TMEM and sB are reused by the next tile
  }
  (void)best;
  tc::cp_wait_all();
  int row = 32 * warp + lane;
  int64_t D = bestD + Ep[(size_t)mt * kTile + row];
  uint64_t packed = bestI == 0x7fffffff ? ~0ull : (((uint64_t)(uint32_t)D << 32) | (uint32_t)bestI);
  out[(size_t)blockIdx.y * mpad + (size_t)mt * kTile + row] = packed;
  __syncthreads();
  if (warp == 0) tc::tmem_free(tm, 256);
}

// full targets of [b, e): flag, per-block count, scan, stable write (ascending slots)
__global__ void k_full_flags(const int32_t* __restrict__ targets, Geo g, int32_t b, int32_t e,
                             int32_t* __restrict__ bc) {
  int i = b + blockIdx.x * 256 + threadIdx.x;
  bool f = false;
  if (i < e) {
    int x, y, t;
    decode(g, targets[i], x, y, t);
    f = full_patch(g, x, y, t);
  }
  int c = __syncthreads_count(f);
  if (threadIdx.x == 0) bc[blockIdx.x] = c;
}
__global__ void k_full_scan(int32_t* bc, int nb, int32_t* total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int32_t run = 0;
    for (int k = 0; k < nb; ++k) {
      int32_t v = bc[k];
      bc[k] = run;
      run += v;
    }
    *total = run;
  }
}
__global__ void k_full_write(const int32_t* __restrict__ targets, Geo g, int32_t b, int32_t e,
                             const int32_t* __restrict__ bc, int32_t* __restrict__ list) {
  int i = b + blockIdx.x * 256 + threadIdx.x;
  bool f = false;
  if (i < e) {
    int x, y, t;
    decode(g, targets[i], x, y, t);
    f = full_patch(g, x, y, t);
  }
  __shared__ int32_t wc[8];
  unsigned bal = __ballot_sync(kFull, f);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wc[w] = __popc(bal);
  __syncthreads();
  int off = bc[blockIdx.x];
  for (int k = 0; k < w; ++k) off += wc[k];
  if (f) list[off + __popc(bal & ((1u << lane) - 1))] = i;
}

// merge the split minima (lexicographic (D, index) = smallest D, then smallest source index)
__global__ void k_bf_merge(const uint64_t* __restrict__ part, int splits, int32_t mpad, int32_t m,
                           const int32_t* __restrict__ list, const int32_t* __restrict__ sources,
                           uint64_t* __restrict__ ee, uint8_t* __restrict__ en) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint64_t best = ~0ull;
  for (int s = 0; s < splits; ++s) best = min(best, part[(size_t)s * mpad + i]);
  int slot = list[i];
  ee[slot] = pack_e((uint32_t)(best >> 32), sources[(uint32_t)best]);
  en[slot] = 125;
}

// border (clipped) targets: the CUDA-core path, restricted to non-full targets
__global__ void k_border_list(const int32_t* __restrict__ targets, Geo g, int32_t b, int32_t e,
                              int32_t* __restrict__ list, int32_t* __restrict__ count) {
  int i = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e) return;
  int x, y, t;
  decode(g, targets[i], x, y, t);
  if (!full_patch(g, x, y, t)) list[atomicAdd(count, 1)] = i;
}

}  // namespace vinp

using namespace vinp;

extern "C" {

size_t vinp_brute_force_tc_ws_bytes(const vinp_level* lv, int32_t b, int32_t e) {
  if (!lv) return 0;
  int64_t m = std::max<int64_t>(0, e - b), mpad = (m + kTile - 1) / kTile * kTile;
  int64_t npad = ((int64_t)lv->n_sources + kTile - 1) / kTile * kTile;
  int64_t nb = (m + 255) / 256 + 1;
  int splits = 64;
  return (size_t)(mpad * kRow + mpad * 8 + npad * kRow + npad * 8 + mpad * 4 * 2 + nb * 4 + 64 +
                  (int64_t)splits * mpad * 8 + 4096);
}

// implemented in ann.cu: CUDA-core exact NN over an explicit slot list
vinp_status vinp_brute_force_list(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm,
                                  const int32_t* list, int32_t n, void* stream);

vinp_status vinp_brute_force_tc(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm, int32_t b,
                                int32_t e, void* ws, size_t ws_bytes, void* stream) {
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
  char* w = (char*)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
  uint8_t* A = (uint8_t*)w; w += mpad * kRow;
  uint8_t* B = (uint8_t*)w; w += npad * kRow;
  int64_t* Ep = (int64_t*)w; w += mpad * 8;
  int64_t* Eq = (int64_t*)w; w += npad * 8;
  int32_t* list = (int32_t*)w; w += mpad * 4;
  int32_t* blist = (int32_t*)w; w += mpad * 4;
  int nb = (int)((m_all + 255) / 256);
  int32_t* bc = (int32_t*)w; w += ((int64_t)nb + 1) * 4;
  int32_t* cnt = (int32_t*)(((uintptr_t)w + 63) & ~(uintptr_t)63); w = (char*)cnt + 64;
  uint64_t* part = (uint64_t*)(((uintptr_t)w + 63) & ~(uintptr_t)63);
  // 1. full targets of [b, e) (ascending) and the border ones
  k_full_flags<<<nb, 256, 0, s>>>(lv->targets, g, b, e, bc);
  k_full_scan<<<1, 32, 0, s>>>(bc, nb, cnt);
  k_full_write<<<nb, 256, 0, s>>>(lv->targets, g, b, e, bc, list);
  cudaMemsetAsync(cnt + 1, 0, 4, s);
  k_border_list<<<nblk(m_all, 256), 256, 0, s>>>(lv->targets, g, b, e, blist, cnt + 1);
  count_launch(4);
  int32_t h[2];
  if (cudaMemcpyAsync(h, cnt, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return check_launch("vinp_brute_force_tc(count)");
  int32_t m = h[0], nborder = h[1];
  int32_t mp = (m + kTile - 1) / kTile * kTile;
  if (m > 0) {
    // 2. im2col of the full targets (by slot -> position) and of all sources
    k_im2col<<<mp, 128, 0, s>>>(lv->vox, g, lv->targets, list, m, mp, prm->lambda, A, Ep);
    k_im2col<<<(int)npad, 128, 0, s>>>(lv->vox, g, lv->sources, nullptr, lv->n_sources, (int)npad, prm->lambda, B, Eq);
    // 3. tensor-core GEMM + exact argmin, N split across CTAs
    int m_tiles = mp / kTile, n_tiles = (int)(npad / kTile);
    int splits = std::max(1, std::min(std::min(64, n_tiles), (2 * 148 + m_tiles - 1) / m_tiles));
    int per = (n_tiles + splits - 1) / splits;
    splits = (n_tiles + per - 1) / per;
    size_t smem = 2 * (size_t)kTile * kRow + kTile * 8;
    cudaFuncSetAttribute(k_bf_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bf_tc<<<dim3(m_tiles, splits), 128, smem, s>>>(A, Ep, B, Eq, n_tiles, per, prm->lambda, mp, part);
    k_bf_merge<<<nblk(m, 256), 256, 0, s>>>(part, splits, mp, m, list, lv->sources, out->e, out->n);
    count_launch(4);
  }
  st = check_launch("vinp_brute_force_tc");
  if (st) return st;
  if (nborder > 0) return vinp_brute_force_list(lv, out, prm, blist, nborder, stream);
  return VINP_OK;
}


vinp_status vinp_tc_gemm_u8(const uint8_t* A, const uint8_t* B, int K, int32_t* C, void* stream) {
  VINP_REQUIRE(A && B && C && K > 0 && K % 32 == 0 && K <= 512, "vinp_tc_gemm_u8: bad arguments");
  size_t smem = 2 * 128 * (size_t)K;
  cudaFuncSetAttribute(k_tc_gemm_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tc_gemm_probe<<<1, 128, smem, S(stream)>>>(A, B, K, C);
  count_launch();
  return check_launch("vinp_tc_gemm_u8");
}

}  // extern "C"
