// align.cu — NEXT #1: dominant affine motion and realignment (Alg. 2; S3.4 P:744-758;
// readings R36-R40 in DESIGN.md).  Compiled with -fmad=false: every fp64 expression is evaluated
// in the written order with no FMA contraction, and the IRLS normal equations are summed exactly
// (int64 of llrint(term * 2^16)), so the result is independent of the thread/block decomposition.
//
//   k_grey0 / k_grey_down  grey-level estimation pyramid of every frame (R36)
//   k_irls                 one 8-CTA cluster per frame pair (n, n+1), one launch per pyramid
//                          level: IRLS with an exact radix-select median of |r| (11-bit digits,
//                          histograms combined over DSMEM) and a redundant per-CTA 6x6 solve
//                          (R37, R38)
//   k_affine_chain         theta_{n,N_m} and inverses (R39), one thread
//   k_align_warp           bilinear warp of every frame to the reference + mask codes (R40)
//   k_unwarp               inverse warp pasted into the original occluded pixels (R40)
#include "common.cuh"

namespace vinp {
namespace {

#ifndef VINP_IRLS_MINB
#define VINP_IRLS_MINB 2
#endif
#ifndef VINP_IRLS_THREADS
#define VINP_IRLS_THREADS 512
#endif
constexpr int kIrlsThreads = VINP_IRLS_THREADS;
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

// R37: warped position of pixel (i, j) and the top-left corner of its bilinear footprint
__device__ __forceinline__ void irls_pos(int W, int H, const double* p, double cx, double cy, double s, int i,
                                         int j, double& X, double& Y, double& xw, double& yw, int& x0,
                                         int& y0) {
  X = ((double)i - cx) / s;
  Y = ((double)j - cy) / s;
  xw = ((p[0] + p[1] * X) + p[2] * Y) + cx;
  yw = ((p[3] + p[4] * X) + p[5] * Y) + cy;
  x0 = (int)floor(xw);
  y0 = (int)floor(yw);
  if (x0 > W - 2) x0 = W - 2;
  if (y0 > H - 2) y0 = H - 2;
}

// R37: a pixel of frame a votes iff unoccluded, its warp lands in [0, W-1] x [0, H-1], and no
// pixel the bilinear sample or its gradient reads in frame b (4x4 block x0-1..x0+2, y0-1..y0+2,
// clamped) is occluded.  Db = that 4x4 dilation of frame b's mask, precomputed (k_mask_dil).
__device__ __forceinline__ bool irls_pixel(const double* Ia, const uint8_t* Ma, const double* Ib,
                                           const uint8_t* Db, int W, int H, const double* p, double cx,
                                           double cy, double s, int i, int j, Pix& o) {
  if (Ma[(int64_t)j * W + i]) return false;
  double X, Y, xw, yw;
  int x0, y0;
  irls_pos(W, H, p, cx, cy, s, i, j, X, Y, xw, yw, x0, y0);
  if (!(xw >= 0.0 && xw <= (double)(W - 1) && yw >= 0.0 && yw <= (double)(H - 1))) return false;
  if (Db[(int64_t)y0 * W + x0]) return false;
  o.fx = xw - (double)x0;
  o.fy = yw - (double)y0;
  o.r = bil(Ib, W, x0, y0, o.fx, o.fy) - Ia[(int64_t)j * W + i];
  o.x0 = x0;
  o.y0 = y0;
  o.X = X;
  o.Y = Y;
  return true;
}

// Db(x, y) = OR of M over columns x-1..x+2 and rows y-1..y+2 (clamped), every frame of a level
__global__ void k_mask_dil(const uint8_t* __restrict__ M, uint8_t* __restrict__ D, int W, int H) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, t = blockIdx.z;
  if (x >= W) return;
  const uint8_t* F = M + (int64_t)t * W * H;
  uint8_t any = 0;
  for (int yy = y - 1; yy <= y + 2; ++yy) {
    int cy_ = yy < 0 ? 0 : (yy > H - 1 ? H - 1 : yy);
    for (int xx = x - 1; xx <= x + 2; ++xx) {
      int cx_ = xx < 0 ? 0 : (xx > W - 1 ? W - 1 : xx);
      any |= F[(int64_t)cy_ * W + cx_];
    }
  }
  D[(int64_t)t * W * H + (int64_t)y * W + x] = any;
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

// exact warp sum of per-lane int64 terms with |v| < 2^40 (the IRLS terms are < 2^32): a signed
// high part and a 16-bit low part, each summed by one REDUX (no partial sum can overflow int32)
__device__ __forceinline__ long long warp_sum_ll(long long v) {
  const int hi = __reduce_add_sync(kFull, (int)(v >> 16));
  const unsigned lo = __reduce_add_sync(kFull, (unsigned)(v & 0xffff));
  return (long long)hi * 65536 + (long long)lo;
}

struct IrlsLevel {
  const double* I;   // [T][W*H]
  const uint8_t* M;  // [T][W*H]
  const uint8_t* D;  // [T][W*H] 4x4 dilation of M
  int W, H;
  double* p;         // [npairs][6] parameter vectors (R37)
  int* status;       // [npairs] 0 / 1 degenerate
  int* iters;        // [npairs] running IRLS iteration count
  uint64_t* keys;    // [npairs][keys_stride] |r| keys, then the odd candidate lists
  uint64_t* cand;    // [npairs][keys_stride] the even candidate lists
  double* rres;      // [npairs][keys_stride] pass-1 residual per pixel (NaN: not voting)
  int64_t keys_stride;
  int max_iter;
  double tol;
};

// R38, one level for pair n: a cluster of kCl CTAs (DSMEM) shares the pixels of the pair.  Every
// cross-CTA quantity (voter count, median digits, the 27 exact sums) is combined by EVERY CTA from
// all ranks' shared memory, so each CTA takes the same decisions and solves the same system
// redundantly (bit-identical: integer sums, same fp64 code) — no broadcast step is needed.
constexpr int kCl = 8;
constexpr int kDigitBits = 11, kBins = 1 << kDigitBits;

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// generic address of the same shared variable in CTA `rank` of the cluster
template <typename Tp>
__device__ __forceinline__ Tp* cl_map(Tp* p, unsigned rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"((uint64_t)p), "r"(rank));
  return reinterpret_cast<Tp*>(out);
}

// histogram of the digit (k >> sh) & dmask of keys with (k & hmask) == prefix: warp-aggregated
__device__ __forceinline__ void hist_add(unsigned* hist, bool act, unsigned d, int lane) {
  unsigned peers = __match_any_sync(kFull, act ? d : 0xffffffffu);
  if (act && lane == __ffs(peers) - 1) atomicAdd(&hist[d], (unsigned)__popc(peers));
}

// Every CTA of the cluster picks the same digit from the summed histograms: the new prefix and
// the rank within it.  Warp 0, 64 bins per lane.
__device__ __forceinline__ void pick_digit(unsigned* hist, int lane, int sh, unsigned long long prefix,
                                           unsigned rank, unsigned long long* s_prefix, unsigned* s_rank) {
  constexpr int kPer = kBins / 32;
  unsigned ls = 0;
  unsigned tb[kPer];
#pragma unroll 4
  for (int q = 0; q < kPer; ++q) {
    unsigned v = 0;
    for (unsigned r = 0; r < kCl; ++r) v += cl_map(hist, r)[lane * kPer + q];
    tb[q] = v;
    ls += v;
  }
  unsigned incl = ls;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    unsigned y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;
  }
  unsigned excl = incl - ls;
  int L = __ffs(__ballot_sync(kFull, rank < incl)) - 1;  // rank < total: some lane holds it
  if (lane == L) {
    unsigned cum = excl;
    int q = 0;
    for (; q < kPer - 1; ++q) {
      if (rank < cum + tb[q]) break;
      cum += tb[q];
    }
    *s_prefix = prefix | ((unsigned long long)(lane * kPer + q) << sh);
    *s_rank = rank - cum;
  }
}

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kIrlsThreads, VINP_IRLS_MINB) k_irls(IrlsLevel a) {
  const int n = blockIdx.x / kCl, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rk = cl_rank();
  if (a.status[n]) return;  // uniform over the cluster
  const int W = a.W, H = a.H;
  const int64_t NP = (int64_t)W * H;
  const double* Ia = a.I + (int64_t)n * NP;
  const double* Ib = Ia + NP;
  const uint8_t* Ma = a.M + (int64_t)n * NP;
  const uint8_t* Db = a.D + (int64_t)(n + 1) * NP;
  // this CTA's contiguous chunk of the pixels; its keys / candidate lists live in the chunk too
  // this CTA's pixels: rows j = rk, rk + kCl, ... (row-interleaved, so occlusions and frame-edge
  // effects spread evenly over the cluster); its keys / candidate lists live in its own region
  const int rows_per = (H + kCl - 1) / kCl;
  const int64_t myN = (int64_t)((H - (int)rk + kCl - 1) / kCl) * W;
  const int64_t c0 = (int64_t)rk * rows_per * W;
  uint64_t* bufA = a.keys + (int64_t)n * a.keys_stride + c0;
  uint64_t* bufB = a.cand + (int64_t)n * a.keys_stride + c0;
  double* rres = a.rres + (int64_t)n * a.keys_stride;
  const double cx = (double)(W - 1) * 0.5, cy = (double)(H - 1) * 0.5;
  const double s = (double)(W > H ? W : H) * 0.5;

  __shared__ double sp[6];
  __shared__ int s_stop, s_status;
  __shared__ unsigned s_nv, s_len;
  __shared__ unsigned hist[kBins];
  __shared__ unsigned long long s_prefix;
  __shared__ unsigned s_rank;
  __shared__ long long red[kIrlsWarps][27];
  __shared__ long long tot[27];
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
    // pass 1: residual keys (bits of |r|) of the voting pixels, compacted into bufA, with the
    // histogram of their first (top 11-bit) digit
    for (int b = tid; b < kBins; b += kIrlsThreads) hist[b] = 0;
    if (tid == 0) s_len = 0;
    __syncthreads();
    for (int64_t base = (tid & ~31); base < myN; base += kIrlsThreads) {
      int64_t id = base + lane;
      bool ok = false;
      unsigned long long key = 0;
      if (id < myN) {
        int jr = (int)(id / W), i = (int)(id - (int64_t)jr * W), j = (int)rk + kCl * jr;
        Pix o;
        ok = irls_pixel(Ia, Ma, Ib, Db, W, H, p, cx, cy, s, i, j, o);
        key = (unsigned long long)__double_as_longlong(fabs(o.r));
        rres[(int64_t)j * W + i] = ok ? o.r : __longlong_as_double(0x7ff8000000000001ll);
      }
      unsigned bal = __ballot_sync(kFull, ok);
      unsigned off = 0;
      if (lane == 0 && bal) off = atomicAdd(&s_len, (unsigned)__popc(bal));
      off = __shfl_sync(kFull, off, 0);
      if (ok) bufA[off + __popc(bal & ((1u << lane) - 1u))] = key;
      hist_add(hist, ok, (unsigned)(key >> (64 - kDigitBits)), lane);
    }
    __syncthreads();
    if (tid == 0) s_nv = s_len;
    cl_sync();
    unsigned nv = 0;
    for (unsigned r = 0; r < kCl; ++r) nv += *cl_map(&s_nv, r);
    if (nv < 12) {
      if (tid == 0) s_status = 1;
      break;  // uniform over the cluster
    }
    // exact lower median: rank (nv-1)/2 by radix select over 11-bit digits (shifts 53..9, then
    // the last 9 bits); each pass filters the previous candidate list by the chosen digit into
    // the other buffer while histogramming the next digit
    unsigned long long prefix = 0ull;
    unsigned rank = (nv - 1) / 2;
    if (warp == 0) pick_digit(hist, lane, 64 - kDigitBits, prefix, rank, &s_prefix, &s_rank);
    cl_sync();  // remote histogram reads done
    prefix = s_prefix;
    rank = s_rank;
    unsigned len = s_len;
    uint64_t* src = bufA;
    uint64_t* dst = bufB;
    for (int shift = 64 - 2 * kDigitBits; shift > -kDigitBits; shift -= kDigitBits) {
      const int sh = shift < 0 ? 0 : shift;
      const int width = shift < 0 ? kDigitBits + shift : kDigitBits;
      const unsigned dmask = (1u << width) - 1u;
      const unsigned long long hmask = ~0ull << (shift + kDigitBits);  // bits fixed by prefix
      __syncthreads();  // everyone has read s_len / s_prefix / s_rank
      for (int b = tid; b < kBins; b += kIrlsThreads) hist[b] = 0;
      if (tid == 0) s_len = 0;
      __syncthreads();
      for (unsigned base = (unsigned)(tid & ~31); base < len; base += kIrlsThreads) {
        unsigned id = base + lane;
        unsigned long long k = id < len ? src[id] : ~0ull;
        bool act = id < len && (k & hmask) == prefix;
        unsigned bal = __ballot_sync(kFull, act);
        unsigned off = 0;
        if (lane == 0 && bal) off = atomicAdd(&s_len, (unsigned)__popc(bal));
        off = __shfl_sync(kFull, off, 0);
        if (act) dst[off + __popc(bal & ((1u << lane) - 1u))] = k;
        hist_add(hist, act, (unsigned)((k >> sh) & dmask), lane);
      }
      cl_sync();  // every rank's histogram and list complete
      if (warp == 0) pick_digit(hist, lane, sh, prefix, rank, &s_prefix, &s_rank);
      cl_sync();  // remote histogram reads done before the next pass clears them
      prefix = s_prefix;
      rank = s_rank;
      len = s_len;
      uint64_t* t_ = src;
      src = dst;
      dst = t_;
    }
    double sigma = 1.4826 * __longlong_as_double((long long)prefix);
    if (sigma < 1e-6) sigma = 1e-6;
    const double c = 4.6851 * sigma;
    // pass 2: exact fixed-point normal equations; each warp reduces its 32 pixels' 27 integer
    // terms with shuffles and lane 0 accumulates the warp's row of `red` (few live registers)
    if (lane < 27) red[warp][lane] = 0;
    __syncwarp();
    for (int64_t base = (tid & ~31); base < myN; base += kIrlsThreads) {
      int64_t id = base + lane;
      bool ok = false;
      double w = 0.0, r = 0.0, J[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      if (id < myN) {
        int jr = (int)(id / W), i = (int)(id - (int64_t)jr * W), j = (int)rk + kCl * jr;
        const double rr = rres[(int64_t)j * W + i];  // pass 1's residual (NaN: not voting)
        if (rr == rr) {
          double u = rr / c;
          if (fabs(u) < 1.0) {
            ok = true;
            double q = 1.0 - u * u;
            w = q * q;
            r = rr;
            Pix o;
            double xw, yw;
            irls_pos(W, H, p, cx, cy, s, i, j, o.X, o.Y, xw, yw, o.x0, o.y0);
            int x0 = o.x0, y0 = o.y0;
            double fx = xw - (double)x0, fy = yw - (double)y0;
            double g00 = gradx(Ib, W, x0, y0), g10 = gradx(Ib, W, x0 + 1, y0);
            double g01 = gradx(Ib, W, x0, y0 + 1), g11 = gradx(Ib, W, x0 + 1, y0 + 1);
            double gx = (1.0 - fy) * ((1.0 - fx) * g00 + fx * g10) + fy * ((1.0 - fx) * g01 + fx * g11);
            g00 = grady(Ib, W, H, x0, y0);
            g10 = grady(Ib, W, H, x0 + 1, y0);
            g01 = grady(Ib, W, H, x0, y0 + 1);
            g11 = grady(Ib, W, H, x0 + 1, y0 + 1);
            double gy = (1.0 - fy) * ((1.0 - fx) * g00 + fx * g10) + fy * ((1.0 - fx) * g01 + fx * g11);
            J[0] = gx; J[1] = gx * o.X; J[2] = gx * o.Y;
            J[3] = gy; J[4] = gy * o.X; J[5] = gy * o.Y;
          }
        }
      }
      if (!__any_sync(kFull, ok)) continue;
      int k = 0;
#pragma unroll
      for (int aa = 0; aa < 6; ++aa) {
        double wa = w * J[aa];
#pragma unroll
        for (int bb = aa; bb < 6; ++bb) {
          long long t = warp_sum_ll(ok ? __double2ll_rn(wa * J[bb] * 65536.0) : 0ll);
          if (lane == 0) red[warp][k] += t;
          ++k;
        }
        long long t = warp_sum_ll(ok ? __double2ll_rn(wa * r * 65536.0) : 0ll);
        if (lane == 0) red[warp][21 + aa] += t;
      }
    }
    __syncthreads();
    if (tid < 27) {
      long long v = 0;
      for (int w = 0; w < kIrlsWarps; ++w) v += red[w][tid];
      tot[tid] = v;
    }
    cl_sync();
    if (tid < 27) {
      long long v = 0;
      for (unsigned r = 0; r < kCl; ++r) v += cl_map(tot, r)[tid];
      red[0][tid] = v;  // cluster total (own red row 0 is free: the warp sums are consumed)
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
    cl_sync();  // tot reads by other ranks done; sp / s_stop published in this CTA
    if (s_stop) break;
  }
  cl_sync();  // no CTA exits while another may still read its shared memory
  if (rk == 0) {
    if (tid < 6) a.p[6 * n + tid] = sp[tid];
    if (tid == 0) {
      a.status[n] = s_status;
      a.iters[n] += iters;
    }
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
  uint8_t* D[8];
  int W[8], H[8];
  uint64_t* keys;
  uint64_t* cand;
  double* rres;
  int64_t stride;
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
    w.D[k] = (uint8_t*)(c ? c + off : nullptr);
    off += al(n);
  }
  w.stride = (int64_t)W * ((H + kCl - 1) / kCl) * kCl;  // >= each level's kCl row-interleaved regions
  w.keys = (uint64_t*)(c ? c + off : nullptr);
  off += al((size_t)w.stride * (T > 1 ? T - 1 : 1) * sizeof(uint64_t));
  w.cand = (uint64_t*)(c ? c + off : nullptr);
  off += al((size_t)w.stride * (T > 1 ? T - 1 : 1) * sizeof(uint64_t));
  w.rres = (double*)(c ? c + off : nullptr);
  off += al((size_t)w.stride * (T > 1 ? T - 1 : 1) * sizeof(double));
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
                                 int max_iter, double tol, int32_t pair_b, int32_t pair_e, double* theta,
                                 int32_t* status, int32_t* iters, void* ws, size_t ws_bytes, void* stream) {
  VINP_NVTX();
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
  for (int k = 0; k < L; ++k) {
    dim3 g((w.W[k] + 127) / 128, w.H[k], T);
    k_mask_dil<<<g, 128, 0, s>>>(w.M[k], w.D[k], w.W[k], w.H[k]);
    count_launch();
  }
  const int p0 = pair_b < 0 ? 0 : pair_b, p1 = (pair_e < 0 || pair_e > T - 1) ? T - 1 : pair_e;
  const int np = p1 - p0;  // pairs [p0, p1): theta/status/iters rows p0.., internal state 0..np-1
  if (np <= 0) return check_launch("vinp_affine_estimate");
  double sc = (double)(w.W[L - 1] > w.H[L - 1] ? w.W[L - 1] : w.H[L - 1]) * 0.5;
  k_affine_init<<<(np + 127) / 128, 128, 0, s>>>(w.p, status + p0, iters + p0, np, sc);
  count_launch();
  for (int k = L - 1; k >= 0; --k) {
    if (k < L - 1) {
      k_level_up<<<(np + 127) / 128, 128, 0, s>>>(w.p, status + p0, np, w.W[k + 1], w.H[k + 1], w.W[k], w.H[k]);
      count_launch();
    }
    const int64_t fk = (int64_t)w.W[k] * w.H[k] * p0;  // first frame of the range at level k
    IrlsLevel a{w.I[k] + fk, w.M[k] + fk, w.D[k] + fk, w.W[k], w.H[k], w.p, status + p0, iters + p0, w.keys,
                w.cand, w.rres, w.stride, max_iter, tol};
    k_irls<<<np * kCl, kIrlsThreads, 0, s>>>(a);
    count_launch();
  }
  k_affine_finish<<<(np + 127) / 128, 128, 0, s>>>(w.p, status + p0, np, W, H, theta + 6 * (int64_t)p0);
  count_launch();
  return check_launch("vinp_affine_estimate");
}

vinp_status vinp_affine_chain(const double* pairs, int T, double* fwd, double* inv, int32_t* err,
                              void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(fwd && inv && err && T >= 1 && (pairs || T == 1), "vinp_affine_chain: bad arguments");
  k_affine_chain<<<1, 1, 0, S(stream)>>>(pairs, T, fwd, inv, err);
  count_launch();
  return check_launch("vinp_affine_chain");
}

vinp_status vinp_align_warp(const uint8_t* rgb, const uint8_t* mask, int W, int H, int T, const double* inv,
                            uint8_t* rgb_out, uint8_t* mask_out, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(rgb && mask && inv && rgb_out && mask_out, "vinp_align_warp: null argument");
  VINP_REQUIRE(W >= 2 && H >= 2 && T >= 1 && H <= 65535 && T <= 65535, "vinp_align_warp: bad sizes");
  dim3 g((W + 127) / 128, H, T);
  k_align_warp<<<g, 128, 0, S(stream)>>>(rgb, mask, W, H, inv, rgb_out, mask_out);
  count_launch();
  return check_launch("vinp_align_warp");
}

vinp_status vinp_unwarp(const uint8_t* rgb_aligned, const uint8_t* rgb_orig, const uint8_t* mask_orig, int W,
                        int H, int T, const double* fwd, uint8_t* out, void* stream) {
  VINP_NVTX();
  VINP_REQUIRE(rgb_aligned && rgb_orig && mask_orig && fwd && out, "vinp_unwarp: null argument");
  VINP_REQUIRE(W >= 2 && H >= 2 && T >= 1 && H <= 65535 && T <= 65535, "vinp_unwarp: bad sizes");
  dim3 g((W + 127) / 128, H, T);
  k_unwarp<<<g, 128, 0, S(stream)>>>(rgb_aligned, rgb_orig, mask_orig, W, H, fwd, out);
  count_launch();
  return check_launch("vinp_unwarp");
}

}  // extern "C"
