// setup.cu — pyramid (a1), texture features (a3), source/target sets (a2), onion layers.
// Each of these is one streaming pass over the level; they run once per inpainting call.
#include <atomic>
#include <string>

#include "common.cuh"

namespace vinp {

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}
void count_launch(int n) { g_launches += (uint64_t)n; }
vinp_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return VINP_E_CUDA;
  }
  return VINP_OK;
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// ------------------------------------------------------------------ a1: pyramid
__global__ void k_level1(const uint8_t* __restrict__ rgb, const uint8_t* __restrict__ mask,
                         uint64_t* __restrict__ vox, uint8_t* __restrict__ flags, int N) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  uint32_t c = (uint32_t)rgb[3 * (int64_t)i] | ((uint32_t)rgb[3 * (int64_t)i + 1] << 8) |
               ((uint32_t)rgb[3 * (int64_t)i + 2] << 16);
  vox[i] = c;
  uint8_t m = mask[i];
  flags[i] = m == 2 ? 8 : (m ? 1 : 0);  // 2 = invalid X (R40), other nonzero = H
}

__device__ __forceinline__ int refl101(int i, int n) {
  if (i < 0) i = -i;
  if (i >= n) i = 2 * (n - 1) - i;
  return min(max(i, 0), n - 1);
}

// masked binomial (1,4,6,4,1)^2 low-pass + even decimation (R17); any-of-2x2 occlusion (R18)
__global__ void k_pyramid_down(const uint64_t* __restrict__ fv, const uint8_t* __restrict__ ff,
                               int W, int H, uint64_t* __restrict__ cv, uint8_t* __restrict__ cf,
                               int Wc, int Hc, int T) {
  int X = blockIdx.x * blockDim.x + threadIdx.x;
  int Y = blockIdx.y * blockDim.y + threadIdx.y;
  int t = blockIdx.z;
  if (X >= Wc || Y >= Hc) return;
  const int b[5] = {1, 4, 6, 4, 1};
  int S = 0, a0 = 0, a1 = 0, a2 = 0;
  int64_t base = (int64_t)t * H * W;
#pragma unroll
  for (int j = -2; j <= 2; ++j) {
    int fy = refl101(2 * Y + j, H);
#pragma unroll
    for (int i = -2; i <= 2; ++i) {
      int fx = refl101(2 * X + i, W);
      int64_t f = base + (int64_t)fy * W + fx;
      if (ff[f] & 1) continue;
      int w = b[i + 2] * b[j + 2];
      uint32_t c = (uint32_t)fv[f];
      S += w;
      a0 += w * (int)(c & 255);
      a1 += w * (int)((c >> 8) & 255);
      a2 += w * (int)((c >> 16) & 255);
    }
  }
  uint32_t out = 0;
  if (S) {
    out = (uint32_t)((2 * a0 + S) / (2 * S)) | ((uint32_t)((2 * a1 + S) / (2 * S)) << 8) |
          ((uint32_t)((2 * a2 + S) / (2 * S)) << 16);
  }
  int any = 0;
  for (int dy = 0; dy < 2; ++dy)
    for (int dx = 0; dx < 2; ++dx) {
      int fx = 2 * X + dx, fy = 2 * Y + dy;
      if (fx < W && fy < H) any |= ff[base + (int64_t)fy * W + fx] & 9;  // H and X: any-of 2x2
    }
  int64_t o = ((int64_t)t * Hc + Y) * Wc + X;
  cv[o] = out;
  cf[o] = (uint8_t)any;
}

__global__ void k_output_rgb(const uint64_t* __restrict__ vox, int64_t N, uint8_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  uint32_t c = (uint32_t)vox[i];
  out[3 * i] = (uint8_t)c;
  out[3 * i + 1] = (uint8_t)(c >> 8);
  out[3 * i + 2] = (uint8_t)(c >> 16);
}

// ------------------------------------------------------------------ a3: texture features
__device__ __forceinline__ int luma(uint64_t w) {  // exact x1000 Rec.601 (R14)
  uint32_t c = (uint32_t)w;
  return 299 * (int)(c & 255) + 587 * (int)((c >> 8) & 255) + 114 * (int)((c >> 16) & 255);
}

// horizontal window sums of masked |dY_x| and |dY_y|: ws[p] = {(sx << 8) | cx, (sy << 8) | cy}
// horizontal window sums of masked |dY_x| and |dY_y|: ws[p] = {(sx << 8) | cx, (sy << 8) | cy}.
// A block owns 128 voxels of a row: the per-position terms (|dY|, valid) of its window range
// [x0 - h, x0 + 127 + h] are computed once into shared memory, then each thread sums 2h + 1 of them
// (the same integer sums as per-voxel loops, in any order).
constexpr int kTexTile = 128, kTexMaxH = 32;
__global__ void __launch_bounds__(kTexTile) k_tex_rows(const uint64_t* __restrict__ vox, const uint8_t* __restrict__ flags,
                                                       int W, int H, int T, int h, uint2* __restrict__ ws) {
  __shared__ uint32_t gx[kTexTile + 2 * kTexMaxH], gy[kTexTile + 2 * kTexMaxH];  // (|dY| << 1) | valid
  const int x0 = blockIdx.x * kTexTile, y = blockIdx.y, t = blockIdx.z;
  const int64_t row = ((int64_t)t * H + y) * W;
  const int ya = refl101(y - 1, H), yb = refl101(y + 1, H);
  const int64_t rowa = ((int64_t)t * H + ya) * W, rowb = ((int64_t)t * H + yb) * W;
  const int n = kTexTile + 2 * h;
  for (int k = threadIdx.x; k < n; k += kTexTile) {
    const int qx = x0 - h + k;
    uint32_t vx = 0, vy = 0;
    if (qx >= 0 && qx < W) {
      const int xa = refl101(qx - 1, W), xb = refl101(qx + 1, W);
      if (!(flags[row + xa] & 1) && !(flags[row + xb] & 1))
        vx = ((uint32_t)abs(luma(vox[row + xb]) - luma(vox[row + xa])) << 1) | 1u;
      if (!(flags[rowa + qx] & 1) && !(flags[rowb + qx] & 1))
        vy = ((uint32_t)abs(luma(vox[rowb + qx]) - luma(vox[rowa + qx])) << 1) | 1u;
    }
    gx[k] = vx;
    gy[k] = vy;
  }
  __syncthreads();
  const int x = x0 + threadIdx.x;
  if (x >= W) return;
  uint32_t sx = 0, cx = 0, sy = 0, cy = 0;
  for (int k = threadIdx.x; k <= threadIdx.x + 2 * h; ++k) {  // qx = x - h .. x + h (outside W: 0)
    sx += gx[k] >> 1;
    cx += gx[k] & 1u;
    sy += gy[k] >> 1;
    cy += gy[k] & 1u;
  }
  ws[row + x] = make_uint2((sx << 8) | cx, (sy << 8) | cy);
}

// vertical window sums -> T_q = floor((S + 500c)/(1000c)) into level-1 texture bytes
// A thread walks kColChunk rows of one column with a running window sum (add the entering row,
// subtract the leaving one: the same exact integer sums as summing the 2h + 1 rows afresh).
constexpr int kColChunk = 64;
__global__ void k_tex_cols(const uint2* __restrict__ ws, int W, int H, int T, int h,
                           uint64_t* __restrict__ vox) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y0 = blockIdx.y * kColChunk, t = blockIdx.z;
  if (x >= W) return;
  const int y1 = min(H, y0 + kColChunk);
  const int64_t col = (int64_t)t * H * W + x;
  uint64_t sx = 0, cx = 0, sy = 0, cy = 0;
  for (int qy = max(0, y0 - h); qy <= min(H - 1, y0 + h); ++qy) {
    uint2 v = ws[col + (int64_t)qy * W];
    sx += v.x >> 8; cx += v.x & 255;
    sy += v.y >> 8; cy += v.y & 255;
  }
  for (int y = y0; y < y1; ++y) {
    if (y > y0) {
      if (y + h < H) {
        uint2 v = ws[col + (int64_t)(y + h) * W];
        sx += v.x >> 8; cx += v.x & 255;
        sy += v.y >> 8; cy += v.y & 255;
      }
      if (y - h - 1 >= 0) {
        uint2 v = ws[col + (int64_t)(y - h - 1) * W];
        sx -= v.x >> 8; cx -= v.x & 255;
        sy -= v.y >> 8; cy -= v.y & 255;
      }
    }
    uint32_t tx = cx ? (uint32_t)((sx + 500 * cx) / (1000 * cx)) : 0;
    uint32_t ty = cy ? (uint32_t)((sy + 500 * cy) / (1000 * cy)) : 0;
    int64_t o = col + (int64_t)y * W;
    uint64_t w = vox[o] & 0xffffffffull;
    vox[o] = w | ((uint64_t)(tx | (ty << 8)) << 32);
  }
}

// Eq. 10 with R16: T^l(x,y,t) = T(2^(l-1) x, 2^(l-1) y, t)
__global__ void k_tex_decimate(const uint64_t* __restrict__ v1, int W1, int H1,
                               uint64_t* __restrict__ vl, int Wl, int Hl, int T, int f) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y;
  int t = blockIdx.z;
  if (x >= Wl) return;
  uint64_t s = v1[((int64_t)t * H1 + (int64_t)f * y) * W1 + (int64_t)f * x];
  int64_t o = ((int64_t)t * Hl + y) * Wl + x;
  vl[o] = (vl[o] & 0xffffffffull) | (s & 0xffffffff00000000ull);
}

// ------------------------------------------------------------------ a2: sets (separable)
// tmp bit0: all 5 neighbours along the axis in bounds and (previous bit0); bit1: any in-bounds
// neighbour with previous bit1.  First pass seeds bit0 = unoccluded, bit1 = occluded.
template <int AXIS, bool FIRST, bool LAST>
__global__ void k_sets_pass(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int W,
                            int H, int T, int* __restrict__ counts) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y;
  int t = blockIdx.z;
  bool ok = x < W;
  int a = 0, b = 0;
  int64_t o = ((int64_t)t * H + y) * W + x;
  if (ok) {
    int c = AXIS == 0 ? x : (AXIS == 1 ? y : t);
    int n = AXIS == 0 ? W : (AXIS == 1 ? H : T);
    int64_t stride = AXIS == 0 ? 1 : (AXIS == 1 ? (int64_t)W : (int64_t)W * H);
    a = 1;
#pragma unroll
    for (int d = -2; d <= 2; ++d) {
      int cc = c + d;
      if (cc < 0 || cc >= n) { a = 0; continue; }
      uint8_t v = in[o + d * stride];
      int va = FIRST ? !(v & 9) : (v & 1);  // D~ seed: neither H nor X
      int vb = FIRST ? (v & 1) : ((v >> 1) & 1);
      a &= va;
      b |= vb;
    }
  }
  if (LAST) {
    // out is flags: keep bit0 (H), set bit1 = D~, bit2 = H~
    if (ok) out[o] = (uint8_t)((out[o] & 9) | (a << 1) | (b << 2));
    int ch = __syncthreads_count(ok && b), cho = __syncthreads_count(ok && a);
    int hh = __syncthreads_count(ok && (out[o] & 1));
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      if (ch) atomicAdd(counts + 0, ch);
      if (hh) atomicAdd(counts + 1, hh);
      if (cho) atomicAdd(counts + 2, cho);
    }
  } else if (ok) {
    out[o] = (uint8_t)(a | (b << 1));
  }
}

// ------------------------------------------------------------------ compaction (sorted lists)
constexpr int kCompT = 256, kCompPer = 8, kCompChunk = kCompT * kCompPer;

__global__ void k_comp_count(const uint8_t* __restrict__ flags, int64_t N, int* __restrict__ bc,
                             int nb) {
  int64_t base = (int64_t)blockIdx.x * kCompChunk;
  int c0 = 0, c1 = 0, c2 = 0;
  for (int k = 0; k < kCompPer; ++k) {
    int64_t i = base + k * kCompT + threadIdx.x;
    if (i < N) {
      uint8_t f = flags[i];
      c0 += (f >> 2) & 1;  // targets H~
      c1 += f & 1;         // holes H
      c2 += (f >> 1) & 1;  // sources D~
    }
  }
  __shared__ int s[3][kCompT / 32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  c0 = __reduce_add_sync(kFull, c0);
  c1 = __reduce_add_sync(kFull, c1);
  c2 = __reduce_add_sync(kFull, c2);
  if (lane == 0) { s[0][w] = c0; s[1][w] = c1; s[2][w] = c2; }
  __syncthreads();
  if (threadIdx.x < 3) {
    int a = 0;
    for (int k = 0; k < kCompT / 32; ++k) a += s[threadIdx.x][k];
    bc[threadIdx.x * nb + blockIdx.x] = a;
  }
}

// exclusive scan of bc[3][nb] in place (one block of 1024 threads per list)
__global__ void k_comp_scan(int* __restrict__ bc, int nb) {
  int* a = bc + (int64_t)blockIdx.x * nb;
  __shared__ int carry;
  __shared__ int wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < nb; base += 1024) {
    int i = base + threadIdx.x;
    int v = i < nb ? a[i] : 0;
    int x = v;
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(kFull, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int s = wsum[lane];
      for (int d = 1; d < 32; d <<= 1) {
        int y = __shfl_up_sync(kFull, s, d);
        if (lane >= d) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    int incl = x + (w ? wsum[w - 1] : 0);
    if (i < nb) a[i] = carry + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += incl;
    __syncthreads();
  }
}

__global__ void k_comp_write(const uint8_t* __restrict__ flags, int64_t N,
                             const int* __restrict__ bc, int nb, int32_t* __restrict__ targets,
                             int32_t* __restrict__ holes, int32_t* __restrict__ sources,
                             int32_t* __restrict__ slot) {
  __shared__ int wpre[3][kCompT / 32];
  __shared__ int run[3];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x < 3) run[threadIdx.x] = bc[threadIdx.x * nb + blockIdx.x];
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kCompChunk;
  for (int k = 0; k < kCompPer; ++k) {
    int64_t i = base + k * kCompT + threadIdx.x;
    uint8_t f = i < N ? flags[i] : 0;
    int pr[3] = {(f >> 2) & 1, f & 1, (f >> 1) & 1};
    unsigned bal[3];
    for (int c = 0; c < 3; ++c) {
      bal[c] = __ballot_sync(kFull, pr[c]);
      if (lane == 0) wpre[c][w] = __popc(bal[c]);
    }
    __syncthreads();
    for (int c = 0; c < 3; ++c) {
      int off = run[c];
      for (int k2 = 0; k2 < w; ++k2) off += wpre[c][k2];
      off += __popc(bal[c] & ((1u << lane) - 1));
      if (pr[c]) {
        if (c == 0) targets[off] = (int32_t)i;
        if (c == 1) holes[off] = (int32_t)i;
        if (c == 2) sources[off] = (int32_t)i;
      }
      if (c == 0 && i < N) slot[i] = pr[0] ? off : -1;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      int a = 0;
      for (int k2 = 0; k2 < kCompT / 32; ++k2) a += wpre[threadIdx.x][k2];
      run[threadIdx.x] += a;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ onion layers (Alg. 3, R22)
__global__ void k_layer_init(const uint8_t* __restrict__ flags, uint8_t* __restrict__ layer,
                             int64_t N, int* __restrict__ remaining) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int occ = i < N ? (flags[i] & 1) : 0;
  if (i < N) layer[i] = occ ? 255 : 0;
  int c = __syncthreads_count(occ);
  if (threadIdx.x == 0 && c) atomicAdd(remaining, c);
}

// layer j = unassigned voxels with an in-bounds 3x3x3 neighbour at layer j-1 (in place is safe:
// this pass only reads the value j-1 and only writes j).
__global__ void k_layer_step(uint8_t* __restrict__ layer, int W, int H, int T, int j,
                             int* __restrict__ remaining) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y;
  int t = blockIdx.z;
  int hit = 0;
  if (x < W) {
    int64_t o = ((int64_t)t * H + y) * W + x;
    if (layer[o] == 255) {
      for (int dt = -1; dt <= 1 && !hit; ++dt)
        for (int dy = -1; dy <= 1 && !hit; ++dy)
          for (int dx = -1; dx <= 1 && !hit; ++dx) {
            int qx = x + dx, qy = y + dy, qt = t + dt;
            if (qx < 0 || qx >= W || qy < 0 || qy >= H || qt < 0 || qt >= T) continue;
            if (layer[((int64_t)qt * H + qy) * W + qx] == j - 1) hit = 1;
          }
      if (hit) layer[o] = (uint8_t)j;
    }
  }
  int c = __syncthreads_count(hit);
  if (threadIdx.x == 0 && c) atomicSub(remaining, c);
}

}  // namespace vinp

using namespace vinp;

extern "C" {

const char* vinp_last_error(void) { return g_err.c_str(); }
int vinp_version(void) { return 1; }
uint64_t vinp_launch_count(void) { return g_launches.load(); }

vinp_status vinp_level_dims(int W, int H, int T, int L, int32_t* dims_out) {
  VINP_NVTX();
  VINP_REQUIRE(dims_out && W >= 1 && H >= 1 && T >= 1 && L >= 1 && L <= 16, "vinp_level_dims: bad arguments");
  if ((int64_t)W * H * T >= (1ll << 31)) {
    set_error("vinp_level_dims: %dx%dx%d voxels exceed the 2^31 limit", W, H, T);
    return VINP_E_UNSUPPORTED;
  }
  for (int l = 0; l < L; ++l) {
    dims_out[3 * l] = W;
    dims_out[3 * l + 1] = H;
    dims_out[3 * l + 2] = T;
    W = (W + 1) / 2;
    H = (H + 1) / 2;
  }
  return VINP_OK;
}

vinp_status vinp_build_pyramid(const uint8_t* rgb, const uint8_t* mask, vinp_level* lv, int L,
                               void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(rgb && mask && lv && L >= 1 && L <= 16, "vinp_build_pyramid: bad arguments");
  for (int l = 0; l < L; ++l) {
    vinp_status st = check_level(&lv[l], "vinp_build_pyramid");
    if (st) return st;
    if (l > 0)
      VINP_REQUIRE(lv[l].W == (lv[l - 1].W + 1) / 2 && lv[l].H == (lv[l - 1].H + 1) / 2 &&
                       lv[l].T == lv[0].T,
                   "vinp_build_pyramid: level %d dims must be ceil-halved", l + 1);
  }
  cudaStream_t s = S(stream);
  int64_t N = (int64_t)lv[0].W * lv[0].H * lv[0].T;
  k_level1<<<nblk(N, 256), 256, 0, s>>>(rgb, mask, lv[0].vox, lv[0].flags, (int)N);
  count_launch();
  for (int l = 1; l < L; ++l) {
    dim3 blk(32, 8);
    dim3 grd(nblk(lv[l].W, 32), nblk(lv[l].H, 8), lv[l].T);
    k_pyramid_down<<<grd, blk, 0, s>>>(lv[l - 1].vox, lv[l - 1].flags, lv[l - 1].W, lv[l - 1].H,
                                       lv[l].vox, lv[l].flags, lv[l].W, lv[l].H, lv[l].T);
    count_launch();
  }
  return check_launch("vinp_build_pyramid");
}

vinp_status vinp_output_rgb(const vinp_level* lv1, uint8_t* out, void* stream) {
  VINP_NVTX();
  vinp_status st = check_level(lv1, "vinp_output_rgb");
  if (st) return st;
  VINP_REQUIRE(out, "vinp_output_rgb: null output");
  int64_t N = (int64_t)lv1->W * lv1->H * lv1->T;
  k_output_rgb<<<nblk(N, 256), 256, 0, S(stream)>>>(lv1->vox, N, out);
  count_launch();
  return check_launch("vinp_output_rgb");
}

size_t vinp_texture_ws_bytes(const vinp_level* lv1) {
  return lv1 ? (size_t)lv1->W * lv1->H * lv1->T * sizeof(uint2) : 0;
}

vinp_status vinp_texture_features(const vinp_params* prm, vinp_level* lv, int L, void* ws,
                                  size_t ws_bytes, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(prm && lv && L >= 1 && L <= 16 && ws, "vinp_texture_features: bad arguments");
  VINP_REQUIRE(ws_bytes >= vinp_texture_ws_bytes(&lv[0]), "vinp_texture_features: ws too small");
  int h = prm->tex_half >= 0 ? prm->tex_half : (L >= 2 ? (1 << (L - 2)) : 1);
  VINP_REQUIRE(h <= 32, "vinp_texture_features: tex_half > 32 unsupported");
  cudaStream_t s = S(stream);
  const vinp_level& a = lv[0];
  k_tex_rows<<<dim3(nblk(a.W, kTexTile), a.H, a.T), kTexTile, 0, s>>>(a.vox, a.flags, a.W, a.H, a.T, h, (uint2*)ws);
  k_tex_cols<<<dim3(nblk(a.W, 128), nblk(a.H, kColChunk), a.T), 128, 0, s>>>((const uint2*)ws, a.W, a.H, a.T, h,
                                                                             a.vox);
  count_launch(2);
  for (int l = 1; l < L; ++l) {
    dim3 g2(nblk(lv[l].W, 128), lv[l].H, lv[l].T);
    k_tex_decimate<<<g2, 128, 0, s>>>(a.vox, a.W, a.H, lv[l].vox, lv[l].W, lv[l].H, lv[l].T, 1 << l);
    count_launch();
  }
  return check_launch("vinp_texture_features");
}

size_t vinp_sets_ws_bytes(const vinp_level* lv1) {
  if (!lv1) return 0;
  int64_t N = (int64_t)lv1->W * lv1->H * lv1->T;
  int64_t nb = (N + kCompChunk - 1) / kCompChunk;
  return (size_t)(2 * N + 64 + 3 * nb * sizeof(int) + 256);
}

vinp_status vinp_build_sets(vinp_level* lv, int L, int32_t* counts_out, void* ws, size_t ws_bytes,
                            void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(lv && L >= 1 && L <= 16 && counts_out && ws, "vinp_build_sets: bad arguments");
  VINP_REQUIRE(ws_bytes >= vinp_sets_ws_bytes(&lv[0]), "vinp_build_sets: ws too small");
  cudaStream_t s = S(stream);
  int64_t N0 = (int64_t)lv[0].W * lv[0].H * lv[0].T;
  uint8_t* t1 = (uint8_t*)ws;
  uint8_t* t2 = t1 + N0;
  int* cnt = (int*)(((uintptr_t)(t2 + N0) + 63) & ~(uintptr_t)63);
  cudaMemsetAsync(cnt, 0, sizeof(int) * 3 * 16, s);
  for (int l = 0; l < L; ++l) {
    vinp_level& a = lv[l];
    dim3 grd(nblk(a.W, 128), a.H, a.T);
    k_sets_pass<0, true, false><<<grd, 128, 0, s>>>(a.flags, t1, a.W, a.H, a.T, nullptr);
    k_sets_pass<1, false, false><<<grd, 128, 0, s>>>(t1, t2, a.W, a.H, a.T, nullptr);
    k_sets_pass<2, false, true><<<grd, 128, 0, s>>>(t2, a.flags, a.W, a.H, a.T, cnt + 3 * l);
    count_launch(3);
  }
  vinp_status st = check_launch("vinp_build_sets");
  if (st) return st;
  int host[48];
  if (cudaMemcpyAsync(host, cnt, sizeof(int) * 3 * L, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return check_launch("vinp_build_sets(sync)");
  for (int i = 0; i < 3 * L; ++i) counts_out[i] = host[i];
  for (int l = 0; l < L; ++l) {
    lv[l].n_targets = host[3 * l];
    lv[l].n_holes = host[3 * l + 1];
    lv[l].n_sources = host[3 * l + 2];
  }
  return VINP_OK;
}

vinp_status vinp_build_lists(vinp_level* lv, int L, void* ws, size_t ws_bytes, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(lv && L >= 1 && L <= 16 && ws, "vinp_build_lists: bad arguments");
  VINP_REQUIRE(ws_bytes >= vinp_sets_ws_bytes(&lv[0]), "vinp_build_lists: ws too small");
  cudaStream_t s = S(stream);
  for (int l = 0; l < L; ++l) {
    vinp_level& a = lv[l];
    VINP_REQUIRE(a.slot && (a.targets || !a.n_targets) && (a.holes || !a.n_holes) &&
                     (a.sources || !a.n_sources),
                 "vinp_build_lists: level %d list buffers missing", l + 1);
    int64_t N = (int64_t)a.W * a.H * a.T;
    int nb = (int)((N + kCompChunk - 1) / kCompChunk);
    int* bc = (int*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    k_comp_count<<<nb, kCompT, 0, s>>>(a.flags, N, bc, nb);
    k_comp_scan<<<3, 1024, 0, s>>>(bc, nb);
    k_comp_write<<<nb, kCompT, 0, s>>>(a.flags, N, bc, nb, a.targets, a.holes, a.sources, a.slot);
    count_launch(3);
  }
  return check_launch("vinp_build_lists");
}

vinp_status vinp_layers(vinp_level* lv, int32_t* n_layers_out, void* ws, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(lv && lv->layer && n_layers_out && ws, "vinp_layers: bad arguments");
  vinp_status st = check_level(lv, "vinp_layers");
  if (st) return st;
  cudaStream_t s = S(stream);
  int64_t N = (int64_t)lv->W * lv->H * lv->T;
  int* rem = (int*)ws;
  cudaMemsetAsync(rem, 0, sizeof(int), s);
  k_layer_init<<<nblk(N, 256), 256, 0, s>>>(lv->flags, lv->layer, N, rem);
  count_launch();
  int j = 0, left = 0;
  cudaMemcpyAsync(&left, rem, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  dim3 grd(nblk(lv->W, 128), lv->H, lv->T);
  while (left > 0) {
    ++j;
    if (j > 254) {
      set_error("vinp_layers: more than 254 onion layers");
      return VINP_E_UNSUPPORTED;
    }
    k_layer_step<<<grd, 128, 0, s>>>(lv->layer, lv->W, lv->H, lv->T, j, rem);
    count_launch();
    cudaMemcpyAsync(&left, rem, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  }
  *n_layers_out = j;
  return check_launch("vinp_layers");
}

}  // extern "C"
