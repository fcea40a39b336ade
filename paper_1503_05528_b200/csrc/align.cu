// align.cu — NEXT #1: dominant affine motion and realignment (Alg. 2; S3.4 P:744-758;
// readings R36-R40 in DESIGN.md).  Compiled with -fmad=false: every fp64 expression is evaluated
// in the written order with no FMA contraction, and the IRLS normal equations are summed exactly
// (int64 of llrint(term * 2^16)), so the result is independent of the thread/block decomposition.
//
//   k_grey0 / k_grey_down  grey-level estimation pyramid of every frame (R36)
//   k_irls                 one CTA per frame pair (n, n+1): coarse-to-fine IRLS with exact
//                          radix-select median of |r| and in-CTA 6x6 solve (R37, R38)
//   k_affine_chain         theta_{n,N_m} and inverses (R39), one thread
//   k_align_warp           bilinear warp of every frame to the reference + mask codes (R40)
//   k_unwarp               inverse warp pasted into the original occluded pixels (R40)
#include "common.cuh"

namespace vinp {
namespace {

constexpr int kIrlsThreads = 512;
constexpr int kIrlsWarps = kIrlsThreads / 32;

__global__ void k_grey0(const uint8_t* __restrict__ rgb, const uint8_t* __restrict__ mask, int64_t N,
                        double* __restrict__ I, uint8_t* __restrict__ M) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int g = 299 * (int)rgb[3 * i] + 587 * (int)rgb[3 * i + 1] + 114 * (int)rgb[3 * i + 2];
  I[i] = (double)g / 1000.0;
  M[i] = mask[i] ? 1 : 0;
}

__global__ void k_grey_down(const double* __restrict__ If, const uint8_t* __restrict__ Mf, int Wf, int Hf,
                            double* __restrict__ Ic, uint8_t* __restrict__ Mc, int Wc, int Hc) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, t = blockIdx.z;
  if (i >= Wc) return;
  const double* F = If + (int64_t)t * Wf * Hf;
  const uint8_t* FM = Mf + (int64_t)t * Wf * Hf;
  int64_t a = (int64_t)(2 * j) * Wf + 2 * i;
  int64_t o = (int64_t)t * Wc * Hc + (int64_t)j * Wc + i;
  Ic[o] = (((F[a] + F[a + 1]) + F[a + Wf]) + F[a + Wf + 1]) * 0.25;
  Mc[o] = FM[a] | FM[a + 1] | FM[a + Wf] | FM[a + Wf + 1];
}

__device__ __forceinline__ double bil(const double* I, int W, int x0, int y0, double fx, double fy) {
  const double* r0 = I + (int64_t)y0 * W + x0;
  const double* r1 = r0 + W;
  return (1.0 - fy) * ((1.0 - fx) * r0[0] + fx * r0[1]) + fy * ((1.0 - fx) * r1[0] + fx * r1[1]);
}
__device__ __forceinline__ double gradx(const double* I, int W, int i, int j) {
  int ip = i + 1 < W ? i + 1 : W - 1, im = i - 1 >= 0 ? i - 1 : 0;
  return (I[(int64_t)j * W + ip] - I[(int64_t)j * W + im]) * 0.5;
}
__device__ __forceinline__ double grady(const double* I, int W, int H, int i, int j) {
  int jp = j + 1 < H ? j + 1 : H - 1, jm = j - 1 >= 0 ? j - 1 : 0;
  return (I[(int64_t)jp * W + i] - I[(int64_t)jm * W + i]) * 0.5;
}

struct Pix {
  double r, fx, fy, X, Y;
  int x0, y0;
};

// R37: a pixel of frame a votes iff unoccluded, its warp lands in [0, W-1] x [0, H-1], and no
// pixel the bilinear sample or its gradient reads in frame b (4x4 block, clamped) is occluded.
__device__ __forceinline__ bool irls_pixel(const double* Ia, const uint8_t* Ma, const double* Ib,
                                           const uint8_t* Mb, int W, int H, const double* p, double cx,
                                           double cy, double s, int i, int j, Pix& o) {
  if (Ma[(int64_t)j * W + i]) return false;
  double X = ((double)i - cx) / s, Y = ((double)j - cy) / s;
  double xw = ((p[0] + p[1] * X) + p[2] * Y) + cx;
  double yw = ((p[3] + p[4] * X) + p[5] * Y) + cy;
  if (!(xw >= 0.0 && xw <= (double)(W - 1) && yw >= 0.0 && yw <= (double)(H - 1))) return false;
  int x0 = (int)floor(xw), y0 = (int)floor(yw);
  if (x0 > W - 2) x0 = W - 2;
  if (y0 > H - 2) y0 = H - 2;
  for (int yy = y0 - 1; yy <= y0 + 2; ++yy) {
    int cy_ = yy < 0 ? 0 : (yy > H - 1 ? H - 1 : yy);
    for (int xx = x0 - 1; xx <= x0 + 2; ++xx) {
      int cx_ = xx < 0 ? 0 : (xx > W - 1 ? W - 1 : xx);
      if (Mb[(int64_t)cy_ * W + cx_]) return false;
    }
  }
  o.fx = xw - (double)x0;
  o.fy = yw - (double)y0;
  o.r = bil(Ib, W, x0, y0, o.fx, o.fy) - Ia[(int64_t)j * W + i];
  o.x0 = x0;
  o.y0 = y0;
  o.X = X;
  o.Y = Y;
  return true;
}

__device__ int solve6(double M[6][7], double* x) {
  double md = 0.0;
  for (int k = 0; k < 6; ++k)
    if (fabs(M[k][k]) > md) md = fabs(M[k][k]);
  for (int k = 0; k < 6; ++k) {
    int pr = k;
    for (int r = k + 1; r < 6; ++r)
      if (fabs(M[r][k]) > fabs(M[pr][k])) pr = r;
    if (pr != k)
      for (int c = 0; c < 7; ++c) {
        double tmp = M[k][c];
        M[k][c] = M[pr][c];
        M[pr][c] = tmp;
      }
    if (!(fabs(M[k][k]) > 1e-9 * md)) return 1;
    for (int r = k + 1; r < 6; ++r) {
      double f = M[r][k] / M[k][k];
      for (int c = k; c < 7; ++c) M[r][c] = M[r][c] - f * M[k][c];
    }
  }
  for (int k = 5; k >= 0; --k) {
    double a = M[k][6];
    for (int c = k + 1; c < 6; ++c) a = a - M[k][c] * x[c];
    x[k] = a / M[k][k];
  }
  return 0;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}

struct IrlsLevel {
  const double* I;   // [T][W*H]
  const uint8_t* M;  // [T][W*H]
  int W, H;
  double* p;         // [npairs][6] parameter vectors (R37)
  int* status;       // [npairs] 0 / 1 degenerate
  int* iters;        // [npairs] running IRLS iteration count
  uint64_t* keys;    // [npairs][keys_stride]
  int64_t keys_stride;
  int max_iter;
  double tol;
};

// R38, one level for pair n = blockIdx.x (frames n, n+1).
__global__ void __launch_bounds__(kIrlsThreads) k_irls(IrlsLevel a) {
  const int n = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.status[n]) return;
  const int W = a.W, H = a.H;
  const int64_t NP = (int64_t)W * H;
  const double* Ia = a.I + (int64_t)n * NP;
  const double* Ib = Ia + NP;
  const uint8_t* Ma = a.M + (int64_t)n * NP;
  const uint8_t* Mb = Ma + NP;
  uint64_t* keys = a.keys + (int64_t)n * a.keys_stride;
  const double cx = (double)(W - 1) * 0.5, cy = (double)(H - 1) * 0.5;
  const double s = (double)(W > H ? W : H) * 0.5;

  __shared__ double sp[6];
  __shared__ int s_stop, s_status;
  __shared__ unsigned s_cnt[kIrlsWarps];
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ unsigned s_rank;
  __shared__ long long red[kIrlsWarps][27];
  if (tid < 6) sp[tid] = a.p[6 * n + tid];
  if (tid == 0) {
    s_stop = 0;
    s_status = 0;
  }
  __syncthreads();
  int iters = 0;
  for (int it = 0; it < a.max_iter; ++it) {
    double p[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) p[k] = sp[k];
    // pass 1: residual keys (bits of |r|; non-voting pixels sort last)
    unsigned cnt = 0;
    for (int64_t id = tid; id < NP; id += kIrlsThreads) {
      int j = (int)(id / W), i = (int)(id - (int64_t)j * W);
      Pix o;
      bool ok = irls_pixel(Ia, Ma, Ib, Mb, W, H, p, cx, cy, s, i, j, o);
      keys[id] = ok ? (uint64_t)__double_as_longlong(fabs(o.r)) : ~0ull;
      cnt += ok;
    }
    cnt = __reduce_add_sync(kFull, cnt);
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    unsigned nv = 0;
    for (int w = 0; w < kIrlsWarps; ++w) nv += s_cnt[w];
    if (nv < 12) {
      if (tid == 0) s_status = 1;
      break;  // uniform
    }
    // exact lower median: rank (nv-1)/2 by 8-bit radix select over the 64-bit keys
    unsigned long long prefix = 0ull;
    unsigned rank = (nv - 1) / 2;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += kIrlsThreads) hist[b] = 0;
      __syncthreads();
      unsigned long long hmask = shift == 56 ? 0ull : (~0ull << (shift + 8));
      for (int64_t base = (int64_t)(tid & ~31); base < NP; base += kIrlsThreads) {
        int64_t id = base + lane;
        unsigned long long k = id < NP ? keys[id] : ~0ull;
        bool act = id < NP && (k & hmask) == prefix;
        unsigned d = act ? (unsigned)((k >> shift) & 255ull) : 256u;
        unsigned peers = __match_any_sync(kFull, d);
        if (act && lane == __ffs(peers) - 1) atomicAdd(&hist[d], (unsigned)__popc(peers));
      }
      __syncthreads();
      if (tid == 0) {
        unsigned cum = 0;
        int d = 0;
        for (; d < 255; ++d) {
          if (rank < cum + hist[d]) break;
          cum += hist[d];
        }
        s_prefix = prefix | ((unsigned long long)d << shift);
        s_rank = rank - cum;
      }
      __syncthreads();
      prefix = s_prefix;
      rank = s_rank;
    }
    double sigma = 1.4826 * __longlong_as_double((long long)prefix);
    if (sigma < 1e-6) sigma = 1e-6;
    const double c = 4.6851 * sigma;
    // pass 2: exact fixed-point normal equations
    long long acc[27];
#pragma unroll
    for (int k = 0; k < 27; ++k) acc[k] = 0;
    for (int64_t id = tid; id < NP; id += kIrlsThreads) {
      int j = (int)(id / W), i = (int)(id - (int64_t)j * W);
      Pix o;
      if (!irls_pixel(Ia, Ma, Ib, Mb, W, H, p, cx, cy, s, i, j, o)) continue;
      double u = o.r / c;
      if (!(fabs(u) < 1.0)) continue;
      double q = 1.0 - u * u;
      double w = q * q;
      int x0 = o.x0, y0 = o.y0;
      double fx = o.fx, fy = o.fy;
      double g00 = gradx(Ib, W, x0, y0), g10 = gradx(Ib, W, x0 + 1, y0);
      double g01 = gradx(Ib, W, x0, y0 + 1), g11 = gradx(Ib, W, x0 + 1, y0 + 1);
      double gx = (1.0 - fy) * ((1.0 - fx) * g00 + fx * g10) + fy * ((1.0 - fx) * g01 + fx * g11);
      g00 = grady(Ib, W, H, x0, y0);
      g10 = grady(Ib, W, H, x0 + 1, y0);
      g01 = grady(Ib, W, H, x0, y0 + 1);
      g11 = grady(Ib, W, H, x0 + 1, y0 + 1);
      double gy = (1.0 - fy) * ((1.0 - fx) * g00 + fx * g10) + fy * ((1.0 - fx) * g01 + fx * g11);
      double J[6] = {gx, gx * o.X, gx * o.Y, gy, gy * o.X, gy * o.Y};
      int k = 0;
#pragma unroll
      for (int aa = 0; aa < 6; ++aa) {
        double wa = w * J[aa];
#pragma unroll
        for (int bb = aa; bb < 6; ++bb) acc[k++] += __double2ll_rn(wa * J[bb] * 65536.0);
        acc[21 + aa] += __double2ll_rn(wa * o.r * 65536.0);
      }
    }
#pragma unroll
    for (int k = 0; k < 27; ++k) {
      long long v = warp_sum_ll(acc[k]);
      if (lane == 0) red[warp][k] = v;
    }
    __syncthreads();
    if (tid < 27) {
      long long v = 0;
      for (int w = 0; w < kIrlsWarps; ++w) v += red[w][tid];
      red[0][tid] = v;
    }
    __syncthreads();
    ++iters;
    if (tid == 0) {
      long long S[6][6], R[6];
      int k = 0;
      for (int aa = 0; aa < 6; ++aa)
        for (int bb = aa; bb < 6; ++bb) S[aa][bb] = red[0][k++];
      for (int aa = 0; aa < 6; ++aa) R[aa] = red[0][21 + aa];
      double Mx[6][7], dp[6];
      for (int aa = 0; aa < 6; ++aa) {
        for (int bb = 0; bb < 6; ++bb) Mx[aa][bb] = (double)(aa <= bb ? S[aa][bb] : S[bb][aa]) / 65536.0;
        Mx[aa][6] = -((double)R[aa] / 65536.0);
      }
      if (solve6(Mx, dp)) {
        s_status = 1;
        s_stop = 1;
      } else {
        double nrm = 0.0;
        for (int aa = 0; aa < 6; ++aa) {
          sp[aa] = sp[aa] + dp[aa];
          nrm = nrm + dp[aa] * dp[aa];
        }
        if (sqrt(nrm) < a.tol) s_stop = 1;
      }
    }
    __syncthreads();
    if (s_stop) break;
  }
  __syncthreads();
  if (tid < 6) a.p[6 * n + tid] = sp[tid];
  if (tid == 0) {
    a.status[n] = s_status;
    a.iters[n] += iters;
  }
}

__global__ void k_affine_init(double* p, int* status, int* iters, int npairs, double s) {
  int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= npairs) return;
  double* q = p + 6 * n;
  q[0] = 0.0; q[1] = s; q[2] = 0.0; q[3] = 0.0; q[4] = 0.0; q[5] = s;
  status[n] = 0;
  iters[n] = 0;
}

// coarse level (Wc, Hc) -> fine (Wf, Hf): (A, b) -> (A, 2b + (I - A) d), d = 2 c_c + 0.5 - c_f
__global__ void k_level_up(double* p, const int* status, int npairs, int Wc, int Hc, int Wf, int Hf) {
  int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= npairs || status[n]) return;
  double* q = p + 6 * n;
  double sc = (double)(Wc > Hc ? Wc : Hc) * 0.5, sf = (double)(Wf > Hf ? Wf : Hf) * 0.5;
  double a11 = q[1] / sc, a12 = q[2] / sc, a21 = q[4] / sc, a22 = q[5] / sc;
  double dx = ((double)(Wc - 1) + 0.5) - (double)(Wf - 1) * 0.5;
  double dy = ((double)(Hc - 1) + 0.5) - (double)(Hf - 1) * 0.5;
  double bx = 2.0 * q[0] + ((dx - a11 * dx) - a12 * dy);
  double by = 2.0 * q[3] + ((dy - a21 * dx) - a22 * dy);
  q[0] = bx; q[1] = a11 * sf; q[2] = a12 * sf;
  q[3] = by; q[4] = a21 * sf; q[5] = a22 * sf;
}

__global__ void k_affine_finish(const double* p, const int* status, int npairs, int W, int H, double* theta) {
  int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= npairs) return;
  const double* q = p + 6 * n;
  double* t = theta + 6 * n;
  if (status[n]) {
    t[0] = 0.0; t[1] = 1.0; t[2] = 0.0; t[3] = 0.0; t[4] = 0.0; t[5] = 1.0;
    return;
  }
  double s0 = (double)(W > H ? W : H) * 0.5, cx = (double)(W - 1) * 0.5, cy = (double)(H - 1) * 0.5;
  double a11 = q[1] / s0, a12 = q[2] / s0, a21 = q[4] / s0, a22 = q[5] / s0;
  t[0] = (q[0] + cx) - (a11 * cx + a12 * cy);
  t[1] = a11; t[2] = a12;
  t[3] = (q[3] + cy) - (a21 * cx + a22 * cy);
  t[4] = a21; t[5] = a22;
}

__device__ void compose(const double* t2, const double* t1, double* out) {
  double r[6];
  r[1] = t2[1] * t1[1] + t2[2] * t1[4];
  r[2] = t2[1] * t1[2] + t2[2] * t1[5];
  r[4] = t2[4] * t1[1] + t2[5] * t1[4];
  r[5] = t2[4] * t1[2] + t2[5] * t1[5];
  r[0] = (t2[1] * t1[0] + t2[2] * t1[3]) + t2[0];
  r[3] = (t2[4] * t1[0] + t2[5] * t1[3]) + t2[3];
  for (int i = 0; i < 6; ++i) out[i] = r[i];
}
__device__ int invert(const double* t, double* out) {
  double det = t[1] * t[5] - t[2] * t[4];
  if (!(fabs(det) > 1e-300)) return 1;
  double i11 = t[5] / det, i12 = -t[2] / det, i21 = -t[4] / det, i22 = t[1] / det;
  double r0 = -(i11 * t[0] + i12 * t[3]);
  double r3 = -(i21 * t[0] + i22 * t[3]);
  out[0] = r0; out[1] = i11; out[2] = i12; out[3] = r3; out[4] = i21; out[5] = i22;
  return 0;
}

// R39 (Alg. 2 second loop), one thread: the chain is a sequential product by definition
__global__ void k_affine_chain(const double* pairs, int T, double* fwd, double* inv, int* err) {
  int m = T / 2 - 1;
  if (m < 0) m = 0;
  int bad = 0;
  double* f = fwd + 6 * m;
  f[0] = 0.0; f[1] = 1.0; f[2] = 0.0; f[3] = 0.0; f[4] = 0.0; f[5] = 1.0;
  for (int n = m - 1; n >= 0; --n) compose(fwd + 6 * (n + 1), pairs + 6 * n, fwd + 6 * n);
  for (int n = m + 1; n < T && !bad; ++n) {
    double pi[6];
    if (invert(pairs + 6 * (n - 1), pi)) bad = 1;
    else compose(fwd + 6 * (n - 1), pi, fwd + 6 * n);
  }
  for (int n = 0; n < T && !bad; ++n)
    if (invert(fwd + 6 * n, inv + 6 * n)) bad = 1;
  *err = bad;
}

// R40: clamp-to-edge bilinear RGB sample, rounded half up; footprint bits of nonzero weight
__device__ __forceinline__ int sample_rgb(const uint8_t* F, int W, int H, double xs, double ys, uint8_t* out,
                                          int& x0, int& y0) {
  double xc = xs >= 0.0 ? (xs <= (double)(W - 1) ? xs : (double)(W - 1)) : 0.0;
  double yc = ys >= 0.0 ? (ys <= (double)(H - 1) ? ys : (double)(H - 1)) : 0.0;
  x0 = (int)floor(xc);
  y0 = (int)floor(yc);
  if (x0 > W - 2) x0 = W - 2;
  if (y0 > H - 2) y0 = H - 2;
  double fx = xc - (double)x0, fy = yc - (double)y0;
  const uint8_t* r0 = F + 3 * ((int64_t)y0 * W + x0);
  const uint8_t* r1 = r0 + 3 * (int64_t)W;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v = (1.0 - fy) * ((1.0 - fx) * (double)r0[c] + fx * (double)r0[3 + c]) +
               fy * ((1.0 - fx) * (double)r1[c] + fx * (double)r1[3 + c]);
    double rv = floor(v + 0.5);
    out[c] = (uint8_t)(rv < 0.0 ? 0 : (rv > 255.0 ? 255 : (int)rv));
  }
  int fp = 0;
  if (fx < 1.0 && fy < 1.0) fp |= 1;
  if (fx > 0.0 && fy < 1.0) fp |= 2;
  if (fx < 1.0 && fy > 0.0) fp |= 4;
  if (fx > 0.0 && fy > 0.0) fp |= 8;
  return fp;
}

__global__ void k_align_warp(const uint8_t* __restrict__ rgb, const uint8_t* __restrict__ mask, int W, int H,
                             const double* __restrict__ inv, uint8_t* __restrict__ rgb_out,
                             uint8_t* __restrict__ mask_out) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, t = blockIdx.z;
  if (x >= W) return;
  const double* q = inv + 6 * t;
  double xs = (q[0] + q[1] * (double)x) + q[2] * (double)y;
  double ys = (q[3] + q[4] * (double)x) + q[5] * (double)y;
  int64_t fb = (int64_t)t * W * H;
  int64_t o = fb + (int64_t)y * W + x;
  uint8_t c[3];
  int x0, y0;
  int fp = sample_rgb(rgb + 3 * fb, W, H, xs, ys, c, x0, y0);
  rgb_out[3 * o] = c[0];
  rgb_out[3 * o + 1] = c[1];
  rgb_out[3 * o + 2] = c[2];
  uint8_t m = 0;
  if (!(xs >= 0.0 && xs <= (double)(W - 1) && ys >= 0.0 && ys <= (double)(H - 1))) {
    m = 2;
  } else {
    const uint8_t* M = mask + fb + (int64_t)y0 * W + x0;
    if (((fp & 1) && M[0]) || ((fp & 2) && M[1]) || ((fp & 4) && M[W]) || ((fp & 8) && M[W + 1])) m = 1;
  }
  mask_out[o] = m;
}

__global__ void k_unwarp(const uint8_t* __restrict__ aligned, const uint8_t* __restrict__ orig,
                         const uint8_t* __restrict__ mask, int W, int H, const double* __restrict__ fwd,
                         uint8_t* __restrict__ out) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, t = blockIdx.z;
  if (x >= W) return;
  int64_t fb = (int64_t)t * W * H;
  int64_t o = fb + (int64_t)y * W + x;
  if (!mask[o]) {
    out[3 * o] = orig[3 * o];
    out[3 * o + 1] = orig[3 * o + 1];
    out[3 * o + 2] = orig[3 * o + 2];
    return;
  }
  const double* q = fwd + 6 * t;
  double xs = (q[0] + q[1] * (double)x) + q[2] * (double)y;
  double ys = (q[3] + q[4] * (double)x) + q[5] * (double)y;
  int x0, y0;
  sample_rgb(aligned + 3 * fb, W, H, xs, ys, out + 3 * o, x0, y0);
}

int est_levels(int W, int H, int levels) {
  int L = levels < 1 ? 1 : levels;
  while (L > 1 && ((W >> (L - 1)) < 8 || (H >> (L - 1)) < 8)) --L;
  return L;
}

inline size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

struct AlignWs {
  double* I[8];
  uint8_t* M[8];
  int W[8], H[8];
  uint64_t* keys;
  double* p;
  size_t bytes;
};

AlignWs carve(void* base, int W, int H, int T, int L) {
  AlignWs w{};
  char* c = (char*)base;
  size_t off = 0;
  for (int k = 0; k < L; ++k) {
    w.W[k] = k ? w.W[k - 1] / 2 : W;
    w.H[k] = k ? w.H[k - 1] / 2 : H;
    size_t n = (size_t)w.W[k] * w.H[k] * T;
    w.I[k] = (double*)(c ? c + off : nullptr);
    off += al(n * sizeof(double));
    w.M[k] = (uint8_t*)(c ? c + off : nullptr);
    off += al(n);
  }
  w.keys = (uint64_t*)(c ? c + off : nullptr);
  off += al((size_t)W * H * (T > 1 ? T - 1 : 1) * sizeof(uint64_t));
  w.p = (double*)(c ? c + off : nullptr);
  off += al((size_t)(T > 1 ? T - 1 : 1) * 6 * sizeof(double));
  w.bytes = off;
  return w;
}

}  // namespace
}  // namespace vinp

using namespace vinp;

extern "C" {

size_t vinp_affine_ws_bytes(int W, int H, int T, int levels) {
  if (W < 2 || H < 2 || T < 1) return 0;
  return carve(nullptr, W, H, T, est_levels(W, H, levels)).bytes;
}

vinp_status vinp_affine_estimate(const uint8_t* rgb, const uint8_t* mask, int W, int H, int T, int levels,
                                 int max_iter, double tol, double* theta, int32_t* status, int32_t* iters,
                                 void* ws, size_t ws_bytes, void* stream) {
  VINP_REQUIRE(rgb && mask && theta && status && iters && ws, "vinp_affine_estimate: null argument");
  VINP_REQUIRE(W >= 2 && H >= 2 && T >= 1 && levels >= 1 && levels <= 8 && max_iter >= 0,
               "vinp_affine_estimate: bad sizes");
  VINP_REQUIRE((int64_t)W * H < (1ll << 31), "vinp_affine_estimate: frame too large");
  int L = est_levels(W, H, levels);
  VINP_REQUIRE(ws_bytes >= vinp_affine_ws_bytes(W, H, T, levels), "vinp_affine_estimate: ws too small");
  if (T < 2) return VINP_OK;
  cudaStream_t s = S(stream);
  AlignWs w = carve(ws, W, H, T, L);
  int64_t N = (int64_t)W * H * T;
  k_grey0<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(rgb, mask, N, w.I[0], w.M[0]);
  count_launch();
  for (int k = 1; k < L; ++k) {
    dim3 g((w.W[k] + 127) / 128, w.H[k], T);
    k_grey_down<<<g, 128, 0, s>>>(w.I[k - 1], w.M[k - 1], w.W[k - 1], w.H[k - 1], w.I[k], w.M[k], w.W[k], w.H[k]);
    count_launch();
  }
  int np = T - 1;
  double sc = (double)(w.W[L - 1] > w.H[L - 1] ? w.W[L - 1] : w.H[L - 1]) * 0.5;
  k_affine_init<<<(np + 127) / 128, 128, 0, s>>>(w.p, status, iters, np, sc);
  count_launch();
  for (int k = L - 1; k >= 0; --k) {
    if (k < L - 1) {
      k_level_up<<<(np + 127) / 128, 128, 0, s>>>(w.p, status, np, w.W[k + 1], w.H[k + 1], w.W[k], w.H[k]);
      count_launch();
    }
    IrlsLevel a{w.I[k], w.M[k], w.W[k], w.H[k], w.p, status, iters, w.keys, (int64_t)W * H, max_iter, tol};
    k_irls<<<np, kIrlsThreads, 0, s>>>(a);
    count_launch();
  }
  k_affine_finish<<<(np + 127) / 128, 128, 0, s>>>(w.p, status, np, W, H, theta);
  count_launch();
  return check_launch("vinp_affine_estimate");
}

vinp_status vinp_affine_chain(const double* pairs, int T, double* fwd, double* inv, int32_t* err,
                              void* stream) {
  VINP_REQUIRE(fwd && inv && err && T >= 1 && (pairs || T == 1), "vinp_affine_chain: bad arguments");
  k_affine_chain<<<1, 1, 0, S(stream)>>>(pairs, T, fwd, inv, err);
  count_launch();
  return check_launch("vinp_affine_chain");
}

vinp_status vinp_align_warp(const uint8_t* rgb, const uint8_t* mask, int W, int H, int T, const double* inv,
                            uint8_t* rgb_out, uint8_t* mask_out, void* stream) {
  VINP_REQUIRE(rgb && mask && inv && rgb_out && mask_out, "vinp_align_warp: null argument");
  VINP_REQUIRE(W >= 2 && H >= 2 && T >= 1 && H <= 65535 && T <= 65535, "vinp_align_warp: bad sizes");
  dim3 g((W + 127) / 128, H, T);
  k_align_warp<<<g, 128, 0, S(stream)>>>(rgb, mask, W, H, inv, rgb_out, mask_out);
  count_launch();
  return check_launch("vinp_align_warp");
}

vinp_status vinp_unwarp(const uint8_t* rgb_aligned, const uint8_t* rgb_orig, const uint8_t* mask_orig, int W,
                        int H, int T, const double* fwd, uint8_t* out, void* stream) {
  VINP_REQUIRE(rgb_aligned && rgb_orig && mask_orig && fwd && out, "vinp_unwarp: null argument");
  VINP_REQUIRE(W >= 2 && H >= 2 && T >= 1 && H <= 65535 && T <= 65535, "vinp_unwarp: bad sizes");
  dim3 g((W + 127) / 128, H, T);
  k_unwarp<<<g, 128, 0, S(stream)>>>(rgb_aligned, rgb_orig, mask_orig, W, H, fwd, out);
  count_launch();
  return check_launch("vinp_unwarp");
}

}  // extern "C"
