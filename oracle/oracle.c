/* oracle.c — plain CPU oracle of the video-inpainting hot path (Newson et al., arXiv 1503.05528).
 *
 * TEST INFRASTRUCTURE ONLY — see oracle.h.  Literal loops over the paper's formulas, in the
 * paper's order and notation; fp64 wherever floating point occurs; no -ffast-math.  The only
 * parallelism is an OpenMP `parallel for` over independent targets inside a Jacobi pass (every
 * pass reads one NNF buffer and writes another), so results do not depend on the thread count.
 *
 * Citations: P:n = PAPER.md line n; R<k> = reading k in DESIGN.md §2.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PR 2 /* patch radius: 5x5x5 patches */

static inline int64_t lin(const or_level* lv, int x, int y, int t) {
  return ((int64_t)t * lv->H + y) * lv->W + x;
}
static inline void coords(const or_level* lv, int64_t p, int* x, int* y, int* t) {
  *x = (int)(p % lv->W);
  *y = (int)((p / lv->W) % lv->H);
  *t = (int)(p / ((int64_t)lv->W * lv->H));
}
static inline int inside(const or_level* lv, int x, int y, int t) {
  return x >= 0 && x < lv->W && y >= 0 && y < lv->H && t >= 0 && t < lv->T;
}

/* ------------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), the counter-based RNG the north_star asks
 * for.  Round: (hi0,lo0)=mulhilo(M0,c0); (hi1,lo1)=mulhilo(M1,c2);
 * c <- (hi1^c1^k0, lo1, hi0^c3^k1, lo0); key bump k += (W0,W1).  Key = (seed lo, seed hi).
 * ---------------------------------------------------------------------------------------- */
void or_philox4x32_10(const uint32_t ctr[4], uint64_t seed, uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Counter layout (R3/R8/R21): c0 = voxel linear index p, c1 = PM iteration k
 * (0 for init/repair), c2 = (level<<24)|(stream<<16)|candidate i, c3 = outer code. */
enum { ST_INIT = 1, ST_RS = 2, ST_REPAIR = 3 };
static void draw(uint32_t p, uint32_t k, int level, int stream, int i, uint32_t oc, uint64_t seed,
                 uint32_t out[4]) {
  uint32_t c[4] = {p, k, ((uint32_t)level << 24) | ((uint32_t)stream << 16) | (uint32_t)i, oc};
  or_philox4x32_10(c, seed, out);
}

/* ------------------------------------------------------------------------------------------
 * a1  Video + occlusion pyramid, Alg. 4; spatial only.  R17: binomial
 * (1,4,6,4,1)^2 in x,y, reflect-101 borders, masked and renormalised over unoccluded fine
 * voxels, value = round-half-up(acc/S) = floor((2acc+S)/(2S)), 0 if S = 0; even-index
 * decimation.  R18: a coarse voxel is occluded iff any of its 2x2 fine voxels is.
 * ---------------------------------------------------------------------------------------- */
static int reflect101(int i, int n) {
  if (i < 0) i = -i;
  if (i >= n) i = 2 * (n - 1) - i;
  if (i < 0) i = 0; /* only for n < 3 */
  if (i >= n) i = n - 1;
  return i;
}

void or_pyramid_down(const uint8_t* rgb, const uint8_t* occ, int W, int H, int T, uint8_t* rgb_c,
                     uint8_t* occ_c) {
  static const int b[5] = {1, 4, 6, 4, 1};
  int Wc = (W + 1) / 2, Hc = (H + 1) / 2;
#pragma omp parallel for
  for (int t = 0; t < T; ++t)
    for (int Y = 0; Y < Hc; ++Y)
      for (int X = 0; X < Wc; ++X) {
        int64_t S = 0, acc[3] = {0, 0, 0};
        for (int j = -2; j <= 2; ++j)
          for (int i = -2; i <= 2; ++i) {
            int fx = reflect101(2 * X + i, W), fy = reflect101(2 * Y + j, H);
            int64_t f = ((int64_t)t * H + fy) * W + fx;
            if (occ[f]) continue;
            int w = b[i + 2] * b[j + 2];
            S += w;
            for (int c = 0; c < 3; ++c) acc[c] += (int64_t)w * rgb[3 * f + c];
          }
        int64_t o = ((int64_t)t * Hc + Y) * Wc + X;
        for (int c = 0; c < 3; ++c) rgb_c[3 * o + c] = S ? (uint8_t)((2 * acc[c] + S) / (2 * S)) : 0;
        int any = 0;
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            int fx = 2 * X + dx, fy = 2 * Y + dy;
            if (fx < W && fy < H && occ[((int64_t)t * H + fy) * W + fx]) any = 1;
          }
        occ_c[o] = (uint8_t)any;
      }
}

/* ------------------------------------------------------------------------------------------
 * a3  Texture features, Eq. 8 P:581-588.  R14: grey = Rec.601 luma in exact x1000 integers,
 * Y = 299R + 587G + 114B; I_x(q) = (Y(q+e_x) - Y(q-e_x))/2 (central difference, reflect-101),
 * counted only if both neighbours are unoccluded.  T_x(p) = mean over valid q in nu(p) of
 * |I_x(q)|/1000; stored as T_q = round(2 T_x) = floor((sum|dY| + 500c)/(1000c)), 0 if c = 0.
 * nu(p) = (2h+1)^2 square clipped to the frame (R15).
 * ---------------------------------------------------------------------------------------- */
void or_texture(const uint8_t* rgb, const uint8_t* occ, int W, int H, int T, int h, uint8_t* tex) {
#pragma omp parallel for
  for (int t = 0; t < T; ++t)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        int64_t sx = 0, sy = 0, cx = 0, cy = 0;
        for (int qy = y - h; qy <= y + h; ++qy)
          for (int qx = x - h; qx <= x + h; ++qx) {
            if (qx < 0 || qx >= W || qy < 0 || qy >= H) continue;
            /* derivative along x at q */
            int xa = reflect101(qx - 1, W), xb = reflect101(qx + 1, W);
            int64_t fa = ((int64_t)t * H + qy) * W + xa, fb = ((int64_t)t * H + qy) * W + xb;
            if (!occ[fa] && !occ[fb]) {
              int64_t Ya = 299 * rgb[3 * fa] + 587 * rgb[3 * fa + 1] + 114 * rgb[3 * fa + 2];
              int64_t Yb = 299 * rgb[3 * fb] + 587 * rgb[3 * fb + 1] + 114 * rgb[3 * fb + 2];
              sx += llabs(Yb - Ya);
              cx += 1;
            }
            /* derivative along y at q */
            int ya = reflect101(qy - 1, H), yb = reflect101(qy + 1, H);
            fa = ((int64_t)t * H + ya) * W + qx;
            fb = ((int64_t)t * H + yb) * W + qx;
            if (!occ[fa] && !occ[fb]) {
              int64_t Ya = 299 * rgb[3 * fa] + 587 * rgb[3 * fa + 1] + 114 * rgb[3 * fa + 2];
              int64_t Yb = 299 * rgb[3 * fb] + 587 * rgb[3 * fb + 1] + 114 * rgb[3 * fb + 2];
              sy += llabs(Yb - Ya);
              cy += 1;
            }
          }
        int64_t o = ((int64_t)t * H + y) * W + x;
        tex[2 * o + 0] = cx ? (uint8_t)((sx + 500 * cx) / (1000 * cx)) : 0;
        tex[2 * o + 1] = cy ? (uint8_t)((sy + 500 * cy) / (1000 * cy)) : 0;
      }
}

/* Eq. 10 P:596-613 with R16: T^l(x,y,t) = T(2^(l-1) x, 2^(l-1) y, t), pure decimation. */
void or_texture_decimate(const uint8_t* tex1, int W1, int H1, int T, int level, int Wl, int Hl,
                         uint8_t* texl) {
  int f = 1 << (level - 1);
  for (int t = 0; t < T; ++t)
    for (int y = 0; y < Hl; ++y)
      for (int x = 0; x < Wl; ++x) {
        int64_t s = ((int64_t)t * H1 + (int64_t)f * y) * W1 + (int64_t)f * x;
        int64_t o = ((int64_t)t * Hl + y) * Wl + x;
        texl[2 * o] = tex1[2 * s];
        texl[2 * o + 1] = tex1[2 * s + 1];
      }
}

/* ------------------------------------------------------------------------------------------
 * a2  Sets.  D~ = {p in D : N_p subset of D}, with N_p required to lie inside Omega;
 * H~ = union over p in H of N_p, clipped to Omega.  Literal neighbourhood loops.
 * ---------------------------------------------------------------------------------------- */
void or_sets(const uint8_t* occ, int W, int H, int T, uint8_t* src, uint8_t* tgt) {
#pragma omp parallel for
  for (int t = 0; t < T; ++t)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        int ok = 1, hit = 0;
        for (int dt = -PR; dt <= PR; ++dt)
          for (int dy = -PR; dy <= PR; ++dy)
            for (int dx = -PR; dx <= PR; ++dx) {
              int qx = x + dx, qy = y + dy, qt = t + dt;
              if (qx < 0 || qx >= W || qy < 0 || qy >= H || qt < 0 || qt >= T) {
                ok = 0;
                continue;
              }
              if (occ[((int64_t)qt * H + qy) * W + qx]) {
                ok = 0;
                hit = 1; /* q in H and p in N_q  <=>  q in N_p */
              }
            }
        int64_t o = ((int64_t)t * H + y) * W + x;
        src[o] = (uint8_t)ok;
        tgt[o] = (uint8_t)hit;
      }
}

/* ------------------------------------------------------------------------------------------
 * Onion layers, Alg. 3, literal: H' <- H; while H' != {}: dH' = H' \ Erode(H',B),
 * B = 3x3x3; layer(dH') = j; H' <- Erode(H',B).  R22: out-of-bounds neighbours count as
 * occluded, so layer(p) = L_inf distance from p to D.  Returns the number of layers.
 * ---------------------------------------------------------------------------------------- */
int or_layers(const uint8_t* occ, int W, int H, int T, uint8_t* layer) {
  int64_t N = (int64_t)W * H * T;
  uint8_t* cur = (uint8_t*)malloc(N);
  uint8_t* ero = (uint8_t*)malloc(N);
  memcpy(cur, occ, N);
  memset(layer, 0, N);
  int j = 0;
  for (;;) {
    int64_t left = 0;
    for (int64_t i = 0; i < N; ++i) left += cur[i];
    if (!left) break;
    ++j;
    if (j > 255) { j = -1; break; }
#pragma omp parallel for
    for (int t = 0; t < T; ++t)
      for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
          int64_t o = ((int64_t)t * H + y) * W + x;
          int keep = cur[o];
          for (int dt = -1; dt <= 1 && keep; ++dt)
            for (int dy = -1; dy <= 1 && keep; ++dy)
              for (int dx = -1; dx <= 1 && keep; ++dx) {
                int qx = x + dx, qy = y + dy, qt = t + dt;
                if (qx < 0 || qx >= W || qy < 0 || qy >= H || qt < 0 || qt >= T) continue;
                if (!cur[((int64_t)qt * H + qy) * W + qx]) keep = 0;
              }
          ero[o] = (uint8_t)keep;
        }
    for (int64_t i = 0; i < N; ++i) {
      if (cur[i] && !ero[i]) layer[i] = (uint8_t)j;
      cur[i] = ero[i];
    }
  }
  free(cur);
  free(ero);
  return j;
}

/* ------------------------------------------------------------------------------------------
 * a4  Patch distance, Eq. 9 P:589-593 with the partial form of Eq. 12 P:809-816 (R23/R24):
 *   D(p,q) = sum_{r in N_p, r in Omega, r in K} [4 ||u(r)-u(r-p+q)||^2 + lambda ||T_q(r)-T_q(r-p+q)||^2]
 *   n      = |N_p cap Omega cap K|,    d^2 = D / (4n).
 * K = Omega when kb < 0, else {r : layer(r) < kb}.  q must be in D~ (full patch inside Omega).
 * ---------------------------------------------------------------------------------------- */
void or_patch_ssd(const or_level* lv, int32_t p, int32_t q, int lambda, int kb, uint32_t* D,
                  uint32_t* n) {
  int px, py, pt, qx, qy, qt;
  coords(lv, p, &px, &py, &pt);
  coords(lv, q, &qx, &qy, &qt);
  uint64_t acc = 0;
  uint32_t cnt = 0;
  for (int dt = -PR; dt <= PR; ++dt)
    for (int dy = -PR; dy <= PR; ++dy)
      for (int dx = -PR; dx <= PR; ++dx) {
        int rx = px + dx, ry = py + dy, rt = pt + dt;
        if (!inside(lv, rx, ry, rt)) continue;
        int64_t r = lin(lv, rx, ry, rt);
        if (kb >= 0 && !(lv->layer[r] < kb)) continue;
        int64_t s = lin(lv, qx + dx, qy + dy, qt + dt);
        int64_t c2 = 0, t2 = 0;
        for (int c = 0; c < 3; ++c) {
          int64_t d = (int64_t)lv->rgb[3 * r + c] - lv->rgb[3 * s + c];
          c2 += d * d;
        }
        for (int c = 0; c < 2; ++c) {
          int64_t d = (int64_t)lv->tex[2 * r + c] - lv->tex[2 * s + c];
          t2 += d * d;
        }
        acc += (uint64_t)(4 * c2 + (int64_t)lambda * t2);
        cnt += 1;
      }
  *D = (uint32_t)acc;
  *n = cnt;
}

/* candidate validity: q = p + v inside Omega and in D~ (Alg. 1 "p+phi(q) in D~"). */
static int valid_source(const or_level* lv, int px, int py, int pt, int dx, int dy, int dt) {
  int qx = px + dx, qy = py + dy, qt = pt + dt;
  if (!inside(lv, qx, qy, qt)) return 0;
  return lv->src[lin(lv, qx, qy, qt)] != 0;
}

static int in_layer(const or_level* lv, int32_t p, int only_layer) {
  return only_layer < 0 || lv->layer[p] == only_layer;
}

/* ------------------------------------------------------------------------------------------
 * a5  NNF initialisation.  Random (Alg. 4; R8): source = sources[(U0*|D~|)>>32]
 * with U0 = Philox(p, 0, (level,INIT,0), outer_code).  D and n are left for evaluate.
 * ---------------------------------------------------------------------------------------- */
int64_t or_nnf_init_random(const or_level* lv, or_nnf* nnf, uint64_t seed, int level,
                           uint32_t outer_code, int32_t b, int32_t e) {
  if (lv->n_sources <= 0) return -1;
  for (int32_t s = b; s < e; ++s) {
    int32_t p = lv->targets[s];
    uint32_t u[4];
    draw((uint32_t)p, 0, level, ST_INIT, 0, outer_code, seed, u);
    int32_t q = lv->sources[((uint64_t)u[0] * (uint64_t)lv->n_sources) >> 32];
    int px, py, pt, qx, qy, qt;
    coords(lv, p, &px, &py, &pt);
    coords(lv, q, &qx, &qy, &qt);
    nnf->dx[s] = qx - px;
    nnf->dy[s] = qy - py;
    nnf->dt[s] = qt - pt;
    nnf->D[s] = 0;
    nnf->n[s] = 0;
  }
  return 0;
}

/* Upsampling (Alg. 4): phi_l(x,y,t) = (2dx, 2dy, dt) of phi_{l+1}(x/2, y/2, t)
 * (nearest neighbour).  R21: a shift that is invalid at the fine level is re-drawn uniformly
 * over D~ with U0 = Philox(p, 0, (level,REPAIR,0), 0). */
void or_nnf_upsample(const or_level* coarse, const or_nnf* cn, const or_level* fine, or_nnf* fn,
                     uint64_t seed, int level, int32_t b, int32_t e) {
  for (int32_t s = b; s < e; ++s) {
    int32_t p = fine->targets[s];
    int px, py, pt;
    coords(fine, p, &px, &py, &pt);
    int64_t cp = lin(coarse, px / 2, py / 2, pt);
    int32_t cs = coarse->slot[cp];
    int ok = 0, dx = 0, dy = 0, dt = 0;
    if (cs >= 0) {
      dx = 2 * cn->dx[cs];
      dy = 2 * cn->dy[cs];
      dt = cn->dt[cs];
      ok = valid_source(fine, px, py, pt, dx, dy, dt);
    }
    if (!ok) {
      uint32_t u[4];
      draw((uint32_t)p, 0, level, ST_REPAIR, 0, 0, seed, u);
      int32_t q = fine->sources[((uint64_t)u[0] * (uint64_t)fine->n_sources) >> 32];
      int qx, qy, qt;
      coords(fine, q, &qx, &qy, &qt);
      dx = qx - px;
      dy = qy - py;
      dt = qt - pt;
    }
    fn->dx[s] = dx;
    fn->dy[s] = dy;
    fn->dt[s] = dt;
    fn->D[s] = 0;
    fn->n[s] = 0;
  }
}

/* Evaluate: (D, n) of the current shift on the current u and K (stale caches forbidden). */
int64_t or_nnf_evaluate(const or_level* lv, or_nnf* nnf, int lambda, int kb, int only_layer,
                        int32_t b, int32_t e) {
  int64_t cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(dynamic, 256)
  for (int32_t s = b; s < e; ++s) {
    int32_t p = lv->targets[s];
    if (!in_layer(lv, p, only_layer)) continue;
    int px, py, pt;
    coords(lv, p, &px, &py, &pt);
    int32_t q = (int32_t)lin(lv, px + nnf->dx[s], py + nnf->dy[s], pt + nnf->dt[s]);
    uint32_t D, n;
    or_patch_ssd(lv, p, q, lambda, kb, &D, &n);
    nnf->D[s] = D;
    nnf->n[s] = (uint8_t)n;
    cnt += 1;
  }
  return cnt;
}

static void copy_entry(const or_nnf* in, or_nnf* out, int32_t s) {
  out->dx[s] = in->dx[s];
  out->dy[s] = in->dy[s];
  out->dt[s] = in->dt[s];
  out->D[s] = in->D[s];
  out->n[s] = in->n[s];
}

/* ------------------------------------------------------------------------------------------
 * a6  Propagation, P:371-386 / Alg. 1, as one Jacobi jump pass (R6): candidates in
 * rank order 0 = incumbent phi_in(p); 1,2,3 = phi_in(p + sign*step*e_x / e_y / e_t) (sign = 0:
 * 1..6 = the -step then the +step neighbours), each only if
 * that neighbour is in Omega and in H~.  A candidate is evaluated only if p+v is in Omega and in
 * D~ (R2) and v differs from the incumbent and from every earlier valid candidate; it replaces the
 * best if its distance is strictly smaller (R25).  Returns the number of evaluated candidates.
 * ---------------------------------------------------------------------------------------- */
int64_t or_propagate(const or_level* lv, const or_nnf* in, or_nnf* out, int lambda, int step,
                     int sign, int kb, int only_layer, int32_t b, int32_t e, const or_nnf* prev,
                     int64_t* stale) {
  int64_t cnt = 0, nst = 0;
#pragma omp parallel for reduction(+ : cnt, nst) schedule(dynamic, 256)
  for (int32_t s = b; s < e; ++s) {
    int32_t p = lv->targets[s];
    copy_entry(in, out, s);
    if (!in_layer(lv, p, only_layer)) continue;
    int px, py, pt;
    coords(lv, p, &px, &py, &pt);
    int seen[7][3];
    int nseen = 0;
    seen[nseen][0] = in->dx[s]; seen[nseen][1] = in->dy[s]; seen[nseen][2] = in->dt[s]; ++nseen;
    uint32_t bestD = in->D[s];
    /* sign = +1 / -1: the 3 neighbours p + sign*step*e_{x,y,t}; sign = 0 ("both", R6): the 6
     * neighbours p - step*e_{x,y,t} then p + step*e_{x,y,t}, in that rank order */
    int nc = sign == 0 ? 6 : 3;
    for (int a = 0; a < nc; ++a) {
      int sg = sign != 0 ? sign : (a < 3 ? -1 : 1);
      int ax = a % 3;
      int rx = px + (ax == 0 ? sg * step : 0);
      int ry = py + (ax == 1 ? sg * step : 0);
      int rt = pt + (ax == 2 ? sg * step : 0);
      if (!inside(lv, rx, ry, rt)) continue;
      int32_t rs = lv->slot[lin(lv, rx, ry, rt)];
      if (rs < 0) continue; /* neighbour not in H~ */
      int vx = in->dx[rs], vy = in->dy[rs], vt = in->dt[rs];
      if (!valid_source(lv, px, py, pt, vx, vy, vt)) continue;
      int dup = 0;
      for (int k = 0; k < nseen; ++k)
        if (seen[k][0] == vx && seen[k][1] == vy && seen[k][2] == vt) dup = 1;
      if (dup) continue;
      seen[nseen][0] = vx; seen[nseen][1] = vy; seen[nseen][2] = vt; ++nseen;
      /* R41 (count only): the neighbour proposes the shift it proposed in the previous pass with
       * this (step, sign) of the same ANN search, `prev` = that pass's input */
      if (prev && prev->dx[rs] == vx && prev->dy[rs] == vy && prev->dt[rs] == vt) nst += 1;
      uint32_t D, n;
      or_patch_ssd(lv, p, (int32_t)lin(lv, px + vx, py + vy, pt + vt), lambda, kb, &D, &n);
      cnt += 1;
      if (D < bestD) {
        bestD = D;
        out->dx[s] = vx; out->dy[s] = vy; out->dt[s] = vt; out->D[s] = D;
      }
    }
  }
  if (stale) *stale = nst;
  return cnt;
}

/* ------------------------------------------------------------------------------------------
 * a7  Random search, Eq. 3 P:393-404 / Alg. 1 P:435-439 (R1, R3, R7): v0 = phi_in(p); for
 * i = 1, 2, ...: R_i = rmax * rho^i by repeated fp64 multiplication, while R_i >= 1;
 * delta_c = (U_c - 2^31) * 2^-31 in [-1,1) from Philox(p, k, (level,RS,i), outer_code);
 * q_i = p + v0 + floor(R_i * delta).  Evaluated iff q_i in Omega and D~, q_i != p + v0 and q_i
 * differs from every earlier valid candidate; strict improvement in candidate order.
 * ---------------------------------------------------------------------------------------- */
int64_t or_random_search(const or_level* lv, const or_nnf* in, or_nnf* out, int lambda,
                         uint64_t seed, double rho, int rmax, int level, uint32_t outer_code,
                         int pm_iter, int kb, int only_layer, int32_t b, int32_t e) {
  int64_t cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(dynamic, 256)
  for (int32_t s = b; s < e; ++s) {
    int32_t p = lv->targets[s];
    copy_entry(in, out, s);
    if (!in_layer(lv, p, only_layer)) continue;
    int px, py, pt;
    coords(lv, p, &px, &py, &pt);
    int v0x = in->dx[s], v0y = in->dy[s], v0t = in->dt[s];
    int seen[64][3];
    int nseen = 0;
    seen[nseen][0] = v0x; seen[nseen][1] = v0y; seen[nseen][2] = v0t; ++nseen;
    uint32_t bestD = in->D[s];
    double R = (double)rmax;
    for (int i = 1; i < 64; ++i) {
      R = R * rho;
      if (!(R >= 1.0)) break;
      uint32_t u[4];
      draw((uint32_t)p, (uint32_t)pm_iter, level, ST_RS, i, outer_code, seed, u);
      int off[3];
      for (int c = 0; c < 3; ++c) {
        double delta = ((double)u[c] - 2147483648.0) * (1.0 / 2147483648.0);
        off[c] = (int)floor(R * delta);
      }
      int vx = v0x + off[0], vy = v0y + off[1], vt = v0t + off[2];
      if (!valid_source(lv, px, py, pt, vx, vy, vt)) continue;
      int dup = 0;
      for (int k = 0; k < nseen; ++k)
        if (seen[k][0] == vx && seen[k][1] == vy && seen[k][2] == vt) dup = 1;
      if (dup) continue;
      seen[nseen][0] = vx; seen[nseen][1] = vy; seen[nseen][2] = vt; ++nseen;
      uint32_t D, n;
      or_patch_ssd(lv, p, (int32_t)lin(lv, px + vx, py + vy, pt + vt), lambda, kb, &D, &n);
      cnt += 1;
      if (D < bestD) {
        bestD = D;
        out->dx[s] = vx; out->dy[s] = vy; out->dt[s] = vt; out->D[s] = D;
      }
    }
  }
  return cnt;
}

/* ------------------------------------------------------------------------------------------
 * a9/a10  Reconstruction.  For p in H (restricted to layer(p) == layer_j when layer_j >= 0), the
 * contributors are C_p = {q in N_p cap Omega} (Eq. 4), or {q in N_p : layer(q) < j}
 * for an onion layer (Eq. 13), in t-major q order.  Each proposes u(p + phi(q)).
 *   WEIGHTED (Eqs. 4-5): d_q^2 = D_q/(4 n_q) compared as exact rationals; sigma_p^2 =
 *     the ceil(0.75 |C_p|)-th smallest (nearest rank, R10); s_q = exp(-d_q^2 / (2 sigma_p^2)) with
 *     a_q = (D_q n_s) / (2 n_q D_s) in fp64.  If sigma_p = 0: mean over the zero-distance
 *     contributors (R11).
 *   UNWEIGHTED (R20): s_q = 1.
 *   BEST_PATCH (Eq. 6, R13): copy from q* = argmin d_q^2, ties -> smallest q.
 * R26: weights are rounded to integer multiples of 2^-36 (llrint(s_q 2^36)) and the sums
 * N = sum w_q c_q, S = sum w_q are exact integers, so the mean N/S does not depend on summation
 * order.  Output fp32 = (float)((double)N / (double)S) (both exact, one rounding each); the
 * working copy is committed by or_commit.  Texture features are reconstructed with the same
 * weights (Eq. 11).
 * ---------------------------------------------------------------------------------------- */
static int key_less(uint32_t Da, uint32_t na, uint32_t Db, uint32_t nb) {
  return (uint64_t)Da * nb < (uint64_t)Db * na;
}

void or_reconstruct(or_level* lv, const or_nnf* nnf, int mode, int layer_j, int32_t hb,
                    int32_t he, float* out_rgb, float* out_tex) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t h = hb; h < he; ++h) {
    int32_t p = lv->holes[h];
    if (layer_j >= 0 && lv->layer[p] != layer_j) continue;
    int px, py, pt;
    coords(lv, p, &px, &py, &pt);
    int32_t cq[125], cs[125];
    int m = 0;
    for (int dt = -PR; dt <= PR; ++dt)
      for (int dy = -PR; dy <= PR; ++dy)
        for (int dx = -PR; dx <= PR; ++dx) {
          int qx = px + dx, qy = py + dy, qt = pt + dt;
          if (!inside(lv, qx, qy, qt)) continue;
          int32_t q = (int32_t)lin(lv, qx, qy, qt);
          if (layer_j >= 0 && !(lv->layer[q] < layer_j)) continue;
          int32_t s = lv->slot[q];
          if (s < 0) continue; /* cannot happen for p in H (q in H~) */
          /* distances are only defined after an evaluate (n > 0); UNWEIGHTED does not use them */
          if (mode != OR_UNWEIGHTED && nnf->n[s] == 0) continue;
          cq[m] = q;
          cs[m] = s;
          ++m;
        }
    int64_t w[125];
    if (m == 0) continue;
    if (mode == OR_BEST_PATCH) {
      int best = 0;
      for (int i = 1; i < m; ++i)
        if (key_less(nnf->D[cs[i]], nnf->n[cs[i]], nnf->D[cs[best]], nnf->n[cs[best]])) best = i;
      for (int i = 0; i < m; ++i) w[i] = (i == best);
    } else if (mode == OR_UNWEIGHTED) {
      for (int i = 0; i < m; ++i) w[i] = 1;
    } else {
      /* nearest-rank percentile: the r-th smallest key, r = ceil(0.75 m) */
      int r = (3 * m + 3) / 4;
      int sig = -1;
      for (int i = 0; i < m && sig < 0; ++i) {
        int less = 0, leq = 0;
        for (int k = 0; k < m; ++k) {
          if (key_less(nnf->D[cs[k]], nnf->n[cs[k]], nnf->D[cs[i]], nnf->n[cs[i]])) ++less;
          if (!key_less(nnf->D[cs[i]], nnf->n[cs[i]], nnf->D[cs[k]], nnf->n[cs[k]])) ++leq;
        }
        if (less < r && leq >= r) sig = i; /* key_i is the r-th smallest value */
      }
      uint32_t Ds = nnf->D[cs[sig]], ns = nnf->n[cs[sig]];
      for (int i = 0; i < m; ++i) {
        uint32_t Dq = nnf->D[cs[i]], nq = nnf->n[cs[i]];
        if (Ds == 0) {
          w[i] = (Dq == 0);
        } else {
          double a = (double)((uint64_t)Dq * ns) / (double)(2 * (uint64_t)nq * Ds);
          w[i] = llrint(exp(-a) * 68719476736.0); /* 2^36 */
        }
      }
    }
    int64_t S = 0, N[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < m; ++i) {
      int32_t s = cs[i];
      int qx, qy, qt;
      coords(lv, cq[i], &qx, &qy, &qt);
      int64_t v = lin(lv, px + nnf->dx[s], py + nnf->dy[s], pt + nnf->dt[s]); /* p + phi(q) */
      S += w[i];
      for (int c = 0; c < 3; ++c) N[c] += w[i] * lv->rgb[3 * v + c];
      for (int c = 0; c < 2; ++c) N[3 + c] += w[i] * lv->tex[2 * v + c];
      (void)qx; (void)qy; (void)qt;
    }
    for (int c = 0; c < 3; ++c) out_rgb[3 * (int64_t)h + c] = (float)((double)N[c] / (double)S);
    for (int c = 0; c < 2; ++c) out_tex[2 * (int64_t)h + c] = (float)((double)N[3 + c] / (double)S);
  }
}

/* Commit reconstructed hole values into the u8 working copy used by the next SSD (R26):
 * floor(x + 0.5) of the fp32 output x (round half up). */
void or_commit(or_level* lv, const float* out_rgb, const float* out_tex, int32_t hb, int32_t he) {
  for (int32_t h = hb; h < he; ++h) {
    int32_t p = lv->holes[h];
    for (int c = 0; c < 3; ++c) lv->rgb[3 * (int64_t)p + c] = (uint8_t)floor((double)out_rgb[3 * (int64_t)h + c] + 0.5);
    for (int c = 0; c < 2; ++c) lv->tex[2 * (int64_t)p + c] = (uint8_t)floor((double)out_tex[2 * (int64_t)h + c] + 0.5);
  }
}

/* Stopping-rule change, Alg. 4 P:988 with R19: sum over hole channels of |a-b|, each term
 * llrint(|a-b| * 2^20) (exact fp64 difference of two floats), summed in int64. */
int64_t or_change_l1(const float* a, const float* b, int64_t n) {
  int64_t s = 0;
  for (int64_t i = 0; i < n; ++i) s += llrint(fabs((double)a[i] - (double)b[i]) * 1048576.0);
  return s;
}

/* The literal P:988 statistic ||u_H - v_H||_2 (stop_rule 1): sum of llrint((a-b)^2 * 2^20); the
 * difference of two floats is exact in fp64 and so is its square (2 x 24 significant bits). */
int64_t or_change_l2(const float* a, const float* b, int64_t n) {
  int64_t s = 0;
  for (int64_t i = 0; i < n; ++i) {
    double d = (double)a[i] - (double)b[i];
    s += llrint(d * d * 1048576.0);
  }
  return s;
}

/* Alg. 4 P:979-988 loop condition "while e > 0.1 and k < k_max" (threshold 0.1,
 * at most 20 iterations; R19 for the norm).  e_fixed is the statistic scaled by 2^20. */
int or_stop(int64_t e_fixed, int64_t n_holes, int k, int max_outer, int stop_rule) {
  if (k >= max_outer) return 1;
  if (stop_rule == 0) /* e_fixed / 2^20 / (3|H|) <= 0.1  <=>  10 e_fixed <= 3|H| 2^20 */
    return 10 * (__int128)e_fixed <= 3 * (__int128)n_holes * 1048576;
  /* sqrt(e_fixed / 2^20) / (3|H|) <= 0.1  <=>  100 e_fixed <= 9 |H|^2 2^20 */
  return 100 * (__int128)e_fixed <= 9 * (__int128)n_holes * n_holes * 1048576;
}

/* Eq. 1 P:286-289 (diagnostic): E = sum_{p in H} d^2(W_p, W_{p+phi(p)}) = sum D/(4n). */
double or_energy(const or_level* lv, const or_nnf* nnf) {
  double E = 0.0;
  for (int32_t h = 0; h < lv->n_holes; ++h) {
    int32_t s = lv->slot[lv->holes[h]];
    if (s >= 0 && nnf->n[s]) E += (double)nnf->D[s] / (4.0 * nnf->n[s]);
  }
  return E;
}

/* Exact NN (the "Matching" step's definition): argmin over q in D~ of D(p,q), K = Omega,
 * scanning D~ in t-major order and keeping the first minimum (ties -> smallest q). */
int64_t or_brute_force(const or_level* lv, or_nnf* out, int lambda, int32_t b, int32_t e) {
  int64_t cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(dynamic, 8)
  for (int32_t s = b; s < e; ++s) {
    int32_t p = lv->targets[s];
    uint32_t bestD = 0xFFFFFFFFu, bestn = 0;
    int32_t bq = -1;
    for (int32_t i = 0; i < lv->n_sources; ++i) {
      uint32_t D, n;
      or_patch_ssd(lv, p, lv->sources[i], lambda, -1, &D, &n);
      cnt += 1;
      if (bq < 0 || D < bestD) {
        bestD = D;
        bestn = n;
        bq = lv->sources[i];
      }
    }
    int px, py, pt, qx, qy, qt;
    coords(lv, p, &px, &py, &pt);
    coords(lv, bq, &qx, &qy, &qt);
    out->dx[s] = qx - px; out->dy[s] = qy - py; out->dt[s] = qt - pt;
    out->D[s] = bestD;
    out->n[s] = (uint8_t)bestn;
  }
  return cnt;
}

/* ------------------------------------------------------------------------------------------
 * Whole pipeline, Alg. 4 P:968-1005 without AlignVideo/UnwarpVideo (NEXT #1).
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  or_level lv;
  or_nnf a, b;
  float *cur_rgb, *cur_tex, *prev_rgb, *prev_tex;
} or_work;

static void build_lists(or_level* lv) {
  int64_t N = (int64_t)lv->W * lv->H * lv->T;
  int32_t nt = 0, nh = 0, ns = 0;
  for (int64_t i = 0; i < N; ++i) {
    nt += lv->tgt[i];
    nh += lv->occ[i];
    ns += lv->src[i];
  }
  lv->targets = (int32_t*)malloc(sizeof(int32_t) * (nt ? nt : 1));
  lv->holes = (int32_t*)malloc(sizeof(int32_t) * (nh ? nh : 1));
  lv->sources = (int32_t*)malloc(sizeof(int32_t) * (ns ? ns : 1));
  lv->slot = (int32_t*)malloc(sizeof(int32_t) * N);
  lv->n_targets = nt; lv->n_holes = nh; lv->n_sources = ns;
  nt = nh = ns = 0;
  for (int64_t i = 0; i < N; ++i) {
    lv->slot[i] = -1;
    if (lv->tgt[i]) { lv->slot[i] = nt; lv->targets[nt++] = (int32_t)i; }
    if (lv->occ[i]) lv->holes[nh++] = (int32_t)i;
    if (lv->src[i]) lv->sources[ns++] = (int32_t)i;
  }
}

static void alloc_nnf(or_nnf* f, int32_t n) {
  size_t k = n ? n : 1;
  f->dx = (int32_t*)calloc(k, 4); f->dy = (int32_t*)calloc(k, 4); f->dt = (int32_t*)calloc(k, 4);
  f->D = (uint32_t*)calloc(k, 4); f->n = (uint8_t*)calloc(k, 1);
}
static void free_nnf(or_nnf* f) { free(f->dx); free(f->dy); free(f->dt); free(f->D); free(f->n); }
static void copy_nnf(const or_nnf* a, or_nnf* b, int32_t n) {
  memcpy(b->dx, a->dx, 4 * (size_t)n); memcpy(b->dy, a->dy, 4 * (size_t)n);
  memcpy(b->dt, a->dt, 4 * (size_t)n); memcpy(b->D, a->D, 4 * (size_t)n);
  memcpy(b->n, a->n, (size_t)n);
}

/* ANN search, Alg. 1 with R3/R5/R6: evaluate; for k = 1..K: for s in steps: propagate(s, sigma_k)
 * with sigma_k = +1 for odd k and -1 for even k (sign_policy 0) or 0 = both directions
 * (sign_policy 1); random_search(k).  Result in w->a. */
static int64_t ann_search(or_work* w, const or_params* prm, int level, uint32_t oc, int kb, int ol,
                          int64_t* stale) {
  or_level* lv = &w->lv;
  int32_t n = lv->n_targets;
  int rmax = lv->W > lv->H ? lv->W : lv->H;
  if (lv->T > rmax) rmax = lv->T;
  int64_t cnt = or_nnf_evaluate(lv, &w->a, prm->lambda, kb, ol, 0, n);
  /* R41 (count only): snap[i][sign+1] = the input of the last propagation pass of this search
   * with step steps[i] and this sign (i = the first index holding that step) */
  or_nnf snap[8][3];
  int have[8][3];
  memset(have, 0, sizeof(have));
  for (int k = 1; k <= prm->pm_iters; ++k) {
    int sign = prm->sign_policy ? 0 : ((k % 2 == 1) ? 1 : -1);
    for (int i = 0; i < prm->n_steps; ++i) {
      int i0 = 0;
      while (prm->steps[i0] != prm->steps[i]) ++i0;
      int h = have[i0][sign + 1];
      or_nnf* sp = &snap[i0][sign + 1];
      int64_t st = 0;
      cnt += or_propagate(lv, &w->a, &w->b, prm->lambda, prm->steps[i], sign, kb, ol, 0, n,
                          h ? sp : NULL, &st);
      if (stale) *stale += st;
      if (!h) {
        sp->dx = (int32_t*)malloc(4 * (size_t)(n ? n : 1));
        sp->dy = (int32_t*)malloc(4 * (size_t)(n ? n : 1));
        sp->dt = (int32_t*)malloc(4 * (size_t)(n ? n : 1));
        have[i0][sign + 1] = 1;
      }
      memcpy(sp->dx, w->a.dx, 4 * (size_t)n);
      memcpy(sp->dy, w->a.dy, 4 * (size_t)n);
      memcpy(sp->dt, w->a.dt, 4 * (size_t)n);
      copy_nnf(&w->b, &w->a, n);
    }
    cnt += or_random_search(lv, &w->a, &w->b, prm->lambda, prm->seed, prm->rho, rmax, level, oc, k,
                            kb, ol, 0, n);
    copy_nnf(&w->b, &w->a, n);
  }
  for (int i = 0; i < 8; ++i)
    for (int g = 0; g < 3; ++g)
      if (have[i][g]) { free(snap[i][g].dx); free(snap[i][g].dy); free(snap[i][g].dt); }
  return cnt;
}

int or_inpaint(const uint8_t* rgb, const uint8_t* occ, int W, int H, int T, const or_params* prm,
               uint8_t* out_rgb, or_stats* st) {
  int L = prm->levels;
  if (L < 1 || L > 16) return 1;
  or_work* w = (or_work*)calloc(L + 1, sizeof(or_work));
  uint8_t* inv[17] = {0};
  memset(st, 0, sizeof(*st));
  /* pyramids: Alg. 4 */
  for (int l = 1; l <= L; ++l) {
    or_level* lv = &w[l].lv;
    lv->W = l == 1 ? W : (w[l - 1].lv.W + 1) / 2;
    lv->H = l == 1 ? H : (w[l - 1].lv.H + 1) / 2;
    lv->T = T;
    int64_t N = (int64_t)lv->W * lv->H * T;
    lv->rgb = (uint8_t*)malloc(3 * N);
    lv->tex = (uint8_t*)malloc(2 * N);
    lv->occ = (uint8_t*)malloc(N);
    lv->src = (uint8_t*)malloc(N);
    lv->tgt = (uint8_t*)malloc(N);
    lv->layer = NULL;
    inv[l] = (uint8_t*)malloc(N);
    if (l == 1) {
      memcpy(lv->rgb, rgb, 3 * N);
      for (int64_t i = 0; i < N; ++i) { /* occ codes: 1 (any nonzero but 2) = H, 2 = X (R40) */
        lv->occ[i] = (uint8_t)(occ[i] != 0 && occ[i] != 2);
        inv[l][i] = (uint8_t)(occ[i] == 2);
      }
    } else {
      or_level* f = &w[l - 1].lv;
      or_pyramid_down(f->rgb, f->occ, f->W, f->H, T, lv->rgb, lv->occ);
      or_mask_down(inv[l - 1], f->W, f->H, T, inv[l]);
    }
  }
  int h = prm->tex_half >= 0 ? prm->tex_half : ((L >= 2 ? (1 << (L - 2)) : 1));
  if (h < 1 && prm->tex_half < 0) h = 1;
  or_texture(w[1].lv.rgb, w[1].lv.occ, W, H, T, h, w[1].lv.tex);
  for (int l = 2; l <= L; ++l)
    or_texture_decimate(w[1].lv.tex, W, H, T, l, w[l].lv.W, w[l].lv.H, w[l].lv.tex);
  for (int l = 1; l <= L; ++l) {
    or_level* lv = &w[l].lv;
    or_sets_x(lv->occ, inv[l], lv->W, lv->H, T, lv->src, lv->tgt);
    build_lists(lv);
    if (lv->n_sources == 0) return 2;
    alloc_nnf(&w[l].a, lv->n_targets);
    alloc_nnf(&w[l].b, lv->n_targets);
    size_t nh = lv->n_holes ? lv->n_holes : 1;
    w[l].cur_rgb = (float*)calloc(3 * nh, 4); w[l].cur_tex = (float*)calloc(2 * nh, 4);
    w[l].prev_rgb = (float*)calloc(3 * nh, 4); w[l].prev_tex = (float*)calloc(2 * nh, 4);
  }
  /* coarsest level: random phi then onion peel (Alg. 3; R22) */
  {
    or_work* c = &w[L];
    or_level* lv = &c->lv;
    int64_t N = (int64_t)lv->W * lv->H * T;
    lv->layer = (uint8_t*)malloc(N);
    int nl = or_layers(lv->occ, lv->W, lv->H, T, lv->layer);
    if (nl < 0) return 3;
    st->onion_layers = nl;
    or_nnf_init_random(lv, &c->a, prm->seed, L, 0, 0, lv->n_targets);
    for (int j = 0; j <= nl; ++j) {
      int kb = j < 1 ? 1 : j;
      st->patch_updates[L - 1] += ann_search(c, prm, L, 0x80000000u | (uint32_t)j, kb, j,
                                             &st->stale[L - 1]);
      if (j >= 1) {
        or_reconstruct(lv, &c->a, OR_WEIGHTED, j, 0, lv->n_holes, c->cur_rgb, c->cur_tex);
        /* commit only layer j (the others are untouched in cur) */
        for (int32_t hh = 0; hh < lv->n_holes; ++hh)
          if (lv->layer[lv->holes[hh]] == j) {
            or_commit(lv, c->cur_rgb, c->cur_tex, hh, hh + 1);
            st->onion_commits += 1;
          }
      }
    }
  }
  /* level loop, Alg. 4 */
  for (int l = L; l >= 1; --l) {
    or_work* c = &w[l];
    or_level* lv = &c->lv;
    int k = 0;
    st->n_holes[l - 1] = lv->n_holes;
    for (;;) {
      memcpy(c->prev_rgb, c->cur_rgb, 12 * (size_t)lv->n_holes);
      memcpy(c->prev_tex, c->cur_tex, 8 * (size_t)lv->n_holes);
      st->patch_updates[l - 1] += ann_search(c, prm, l, (uint32_t)k, -1, -1, &st->stale[l - 1]);
      or_reconstruct(lv, &c->a, OR_WEIGHTED, -1, 0, lv->n_holes, c->cur_rgb, c->cur_tex);
      or_commit(lv, c->cur_rgb, c->cur_tex, 0, lv->n_holes);
      int64_t e = prm->stop_rule == 1 ? or_change_l2(c->cur_rgb, c->prev_rgb, 3 * (int64_t)lv->n_holes)
                                       : or_change_l1(c->cur_rgb, c->prev_rgb, 3 * (int64_t)lv->n_holes);
      if (k < 32) st->change_fixed[l - 1][k] = e;
      ++k;
      if (prm->fixed_outer > 0) {
        if (k >= prm->fixed_outer) break;
      } else if (or_stop(e, lv->n_holes, k, prm->max_outer, prm->stop_rule)) {
        break;
      }
    }
    st->outer_iters[l - 1] = k;
    if (l == 1) {
      or_reconstruct(lv, &c->a, OR_BEST_PATCH, -1, 0, lv->n_holes, c->cur_rgb, c->cur_tex);
      or_commit(lv, c->cur_rgb, c->cur_tex, 0, lv->n_holes);
    } else {
      or_work* f = &w[l - 1];
      or_nnf_upsample(lv, &c->a, &f->lv, &f->a, prm->seed, l - 1, 0, f->lv.n_targets);
      or_reconstruct(&f->lv, &f->a, OR_UNWEIGHTED, -1, 0, f->lv.n_holes, f->cur_rgb, f->cur_tex);
      or_commit(&f->lv, f->cur_rgb, f->cur_tex, 0, f->lv.n_holes);
    }
  }
  memcpy(out_rgb, w[1].lv.rgb, 3 * (size_t)W * H * T);
  for (int l = 1; l <= L; ++l) {
    or_level* lv = &w[l].lv;
    free(lv->rgb); free(lv->tex); free(lv->occ); free(lv->src); free(lv->tgt); free(lv->layer);
    free(inv[l]);
    free(lv->slot); free(lv->targets); free(lv->holes); free(lv->sources);
    free_nnf(&w[l].a); free_nnf(&w[l].b);
    free(w[l].cur_rgb); free(w[l].cur_tex); free(w[l].prev_rgb); free(w[l].prev_tex);
  }
  free(w);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * App. B: W, V i.i.d. N(mu, sigma^2)^N, Z = mu.  With X = (W-mu)/sigma,
 * Y = (V-mu)/sigma:  ||W-V||^2 < ||W-Z||^2  <=>  ||Y||^2 < 2 <X,Y>, and <X,Y> | Y ~ N(0, ||Y||^2),
 * so P_N = E[Q(||Y|| / 2)], ||Y||^2 ~ chi2_N.  Integral over s = ||Y|| by composite Simpson on
 * [0, sqrt(N) + 40] (the chi density of s is negligible beyond), in log space.
 * ---------------------------------------------------------------------------------------- */
double or_ambiguity_exact(int N) {
  const int n = 400000;
  double smax = sqrt((double)N) + 40.0, h = smax / n, acc = 0.0;
  /* chi density of s = ||Y||: s^(N-1) e^(-s^2/2) / (2^(N/2-1) Gamma(N/2)) */
  double lc = -(N / 2.0 - 1.0) * log(2.0) - lgamma(N / 2.0);
  for (int i = 0; i <= n; ++i) {
    double s = i * h;
    double f;
    if (s > 0)
      f = exp(lc + (N - 1) * log(s) - s * s / 2.0);
    else
      f = N == 1 ? exp(lc) : 0.0;
    f *= 0.5 * erfc(s / 2.0 / sqrt(2.0)); /* Q(s/2) */
    double w = (i == 0 || i == n) ? 1.0 : ((i & 1) ? 4.0 : 2.0);
    acc += w * f;
  }
  return acc * h / 3.0;
}

/* The paper's simulation (Table 2 caption): per trial draw W, V ~ N(0, sigma^2)^N, count
 * sum (W-V)^2 < sum W^2.  Normals: Box-Muller on Philox words (u1 = (U0 + 0.5) 2^-32,
 * u2 = U1 2^-32 -> two normals; U2, U3 -> two more), component pair k = components 4k..4k+3. */
int64_t or_ambiguity_mc(int N, double sigma, uint64_t seed, uint64_t trial0, uint64_t n_trials) {
  int64_t hits = 0;
#pragma omp parallel for reduction(+ : hits) schedule(static, 4096)
  for (int64_t tr = 0; tr < (int64_t)n_trials; ++tr) {
    uint64_t t = trial0 + (uint64_t)tr;
    double a = 0.0, b = 0.0, z[4];
    /* 2N normals, 4 per Philox call; W_c uses normal 2c, V_c normal 2c + 1 */
    int nn = 2 * N;
    double w = 0.0;
    for (int k = 0; k < (nn + 3) / 4; ++k) {
      uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32), (4u << 16) | (uint32_t)k, 0u}, u[4];
      or_philox4x32_10(ctr, seed, u);
      double r1 = sqrt(-2.0 * log(((double)u[0] + 0.5) / 4294967296.0));
      double r2 = sqrt(-2.0 * log(((double)u[2] + 0.5) / 4294967296.0));
      double th1 = 2.0 * 3.14159265358979323846 * ((double)u[1] / 4294967296.0);
      double th2 = 2.0 * 3.14159265358979323846 * ((double)u[3] / 4294967296.0);
      z[0] = r1 * cos(th1); z[1] = r1 * sin(th1); z[2] = r2 * cos(th2); z[3] = r2 * sin(th2);
      for (int j = 0; j < 4; ++j) {
        int idx = 4 * k + j;
        if (idx >= nn) break;
        if ((idx & 1) == 0) {
          w = sigma * z[j];          /* W_c - mu, c = idx / 2 */
        } else {
          double v = sigma * z[j];   /* V_c - mu */
          a += (w - v) * (w - v);
          b += w * w;
        }
      }
    }
    hits += (a < b);
  }
  return hits;
}

/* ------------------------------------------------------------------------------------------
 * NEXT #2: the paper's sequential ANN search, Alg. 1 P:411-443 as printed (with R1, R2, R3, R7).
 * ---------------------------------------------------------------------------------------- */
static int64_t seq_try(const or_level* lv, or_nnf* f, int32_t s, int32_t p, int px, int py, int pt,
                       int vx, int vy, int vt, int lambda, int (*seen)[3], int* nseen) {
  if (!valid_source(lv, px, py, pt, vx, vy, vt)) return 0;
  for (int k = 0; k < *nseen; ++k)
    if (seen[k][0] == vx && seen[k][1] == vy && seen[k][2] == vt) return 0;
  seen[*nseen][0] = vx; seen[*nseen][1] = vy; seen[*nseen][2] = vt; ++*nseen;
  uint32_t D, n;
  or_patch_ssd(lv, p, (int32_t)lin(lv, px + vx, py + vy, pt + vt), lambda, -1, &D, &n);
  if (D < f->D[s]) {
    f->dx[s] = vx; f->dy[s] = vy; f->dt[s] = vt; f->D[s] = D;
  }
  return 1;
}

int64_t or_ann_search_sequential(const or_level* lv, or_nnf* f, int lambda, uint64_t seed,
                                 double rho, int rmax, int level, uint32_t outer_code, int K) {
  int32_t nt = lv->n_targets;
  int64_t cnt = or_nnf_evaluate(lv, f, lambda, -1, -1, 0, nt);
  for (int k = 1; k <= K; ++k) {
    int fwd = (k % 2 == 0);          /* Alg. 1: k even -> forward scan, p - e_*; odd -> reverse, p + e_* */
    int sg = fwd ? -1 : 1;
    for (int32_t i = 0; i < nt; ++i) {
      int32_t s = fwd ? i : nt - 1 - i;
      int32_t p = lv->targets[s];
      int px, py, pt;
      coords(lv, p, &px, &py, &pt);
      int seen[4][3], nseen = 0;
      seen[0][0] = f->dx[s]; seen[0][1] = f->dy[s]; seen[0][2] = f->dt[s]; nseen = 1;
      for (int a = 0; a < 3; ++a) {
        int rx = px + (a == 0 ? sg : 0), ry = py + (a == 1 ? sg : 0), rt = pt + (a == 2 ? sg : 0);
        if (!inside(lv, rx, ry, rt)) continue;
        int32_t rs = lv->slot[lin(lv, rx, ry, rt)];
        if (rs < 0) continue;
        /* the neighbour's CURRENT shift: already updated in this scan if it precedes p */
        cnt += seq_try(lv, f, s, p, px, py, pt, f->dx[rs], f->dy[rs], f->dt[rs], lambda, seen, &nseen);
      }
    }
    for (int32_t s = 0; s < nt; ++s) {  /* random search, lexicographic order (Alg. 1) */
      int32_t p = lv->targets[s];
      int px, py, pt;
      coords(lv, p, &px, &py, &pt);
      int v0x = f->dx[s], v0y = f->dy[s], v0t = f->dt[s];
      int seen[64][3], nseen = 1;
      seen[0][0] = v0x; seen[0][1] = v0y; seen[0][2] = v0t;
      double R = (double)rmax;
      for (int i = 1; i < 64; ++i) {
        R = R * rho;
        if (!(R >= 1.0)) break;
        uint32_t u[4];
        draw((uint32_t)p, (uint32_t)k, level, ST_RS, i, outer_code, seed, u);
        int off[3];
        for (int c = 0; c < 3; ++c)
          off[c] = (int)floor(R * (((double)u[c] - 2147483648.0) * (1.0 / 2147483648.0)));
        cnt += seq_try(lv, f, s, p, px, py, pt, v0x + off[0], v0y + off[1], v0t + off[2], lambda, seen,
                       &nseen);
      }
    }
  }
  return cnt;
}

/* ==========================================================================================
 * a2 with the invalid set X of a realigned video (R40, S3.4 P:752-753 "the occlusion H is
 * obviously also realigned"; "pixels whose source falls outside the original frame
 * are flagged invalid (excluded from D~)").  Literal neighbourhood loops as or_sets.
 * ======================================================================================== */
void or_sets_x(const uint8_t* occ, const uint8_t* inv, int W, int H, int T, uint8_t* src,
               uint8_t* tgt) {
#pragma omp parallel for
  for (int t = 0; t < T; ++t)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        int ok = 1, hit = 0;
        for (int dt = -PR; dt <= PR; ++dt)
          for (int dy = -PR; dy <= PR; ++dy)
            for (int dx = -PR; dx <= PR; ++dx) {
              int qx = x + dx, qy = y + dy, qt = t + dt;
              if (qx < 0 || qx >= W || qy < 0 || qy >= H || qt < 0 || qt >= T) {
                ok = 0;
                continue;
              }
              int64_t q = ((int64_t)qt * H + qy) * W + qx;
              if (occ[q]) {
                ok = 0;
                hit = 1;
              }
              if (inv && inv[q]) ok = 0;
            }
        int64_t o = ((int64_t)t * H + y) * W + x;
        src[o] = (uint8_t)ok;
        tgt[o] = (uint8_t)hit;
      }
}

void or_mask_down(const uint8_t* m, int W, int H, int T, uint8_t* mc) {
  int Wc = (W + 1) / 2, Hc = (H + 1) / 2;
  for (int t = 0; t < T; ++t)
    for (int Y = 0; Y < Hc; ++Y)
      for (int X = 0; X < Wc; ++X) {
        int any = 0;
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            int fx = 2 * X + dx, fy = 2 * Y + dy;
            if (fx < W && fy < H && m[((int64_t)t * H + fy) * W + fx]) any = 1;
          }
        mc[((int64_t)t * Hc + Y) * Wc + X] = (uint8_t)any;
      }
}

/* ==========================================================================================
 * NEXT #1 — Alg. 2: EstimateAffineMotion(u_n, u_{n+1}) for n = 1..N_f-1, the
 * chain theta_{n,N_m}, AffineWarp; S3.4: Odobez-Bouthemy robust dominant affine
 * motion, "linear interpolation" for the realigned colours, realigned occlusion, inverse
 * transformation and paste into the original occluded area after inpainting.
 * The paper names the estimator only by citation; R36-R38 fix it, after
 * robust penalty of the brightness-constancy residual, IRLS on the linearised
 * residual, 3-level coarse-to-fine, Tukey biweight with MAD scale, <= 20 iterations per level
 * or update norm < 1e-4.  Everything is fp64 written out in a fixed operation order (no FMA
 * contraction: the library is built with -ffp-contract=off) and the normal equations are summed
 * exactly in 2^-16 fixed point, so the GPU's parallel sums reproduce them bit for bit.
 * ======================================================================================== */
void or_affine_compose(const double* t2, const double* t1, double* out) {
  /* (A2, b2) o (A1, b1) = (A2 A1, A2 b1 + b2) */
  double r[6];
  r[1] = t2[1] * t1[1] + t2[2] * t1[4];
  r[2] = t2[1] * t1[2] + t2[2] * t1[5];
  r[4] = t2[4] * t1[1] + t2[5] * t1[4];
  r[5] = t2[4] * t1[2] + t2[5] * t1[5];
  r[0] = (t2[1] * t1[0] + t2[2] * t1[3]) + t2[0];
  r[3] = (t2[4] * t1[0] + t2[5] * t1[3]) + t2[3];
  for (int i = 0; i < 6; ++i) out[i] = r[i];
}

int or_affine_invert(const double* t, double* out) {
  double det = t[1] * t[5] - t[2] * t[4];
  if (!(fabs(det) > 1e-300)) return 1;
  double i11 = t[5] / det, i12 = -t[2] / det, i21 = -t[4] / det, i22 = t[1] / det;
  double r0 = -(i11 * t[0] + i12 * t[3]);
  double r3 = -(i21 * t[0] + i22 * t[3]);
  out[0] = r0; out[1] = i11; out[2] = i12; out[3] = r3; out[4] = i21; out[5] = i22;
  return 0;
}

/* R36: grey level I = (299 R + 587 G + 114 B) / 1000 (exact integer numerator, one division);
 * estimation pyramid: level k = 2x2 box mean of level k-1 on floor(W/2) x floor(H/2), excluded
 * (occluded) if any of the 4 is; the number of levels is reduced while the coarsest would be
 * smaller than 8 pixels on a side. */
typedef struct {
  int W, H;
  double* I;
  uint8_t* M;
} or_grey;

static void grey_pyr(const uint8_t* rgb, const uint8_t* occ, int W, int H, int L, or_grey* P) {
  P[0].W = W; P[0].H = H;
  P[0].I = (double*)malloc(sizeof(double) * W * H);
  P[0].M = (uint8_t*)malloc((size_t)W * H);
  for (int64_t i = 0; i < (int64_t)W * H; ++i) {
    int g = 299 * rgb[3 * i] + 587 * rgb[3 * i + 1] + 114 * rgb[3 * i + 2];
    P[0].I[i] = (double)g / 1000.0;
    P[0].M[i] = (uint8_t)(occ && occ[i] ? 1 : 0);
  }
  for (int k = 1; k < L; ++k) {
    int Wk = P[k - 1].W / 2, Hk = P[k - 1].H / 2, Wf = P[k - 1].W;
    P[k].W = Wk; P[k].H = Hk;
    P[k].I = (double*)malloc(sizeof(double) * Wk * Hk);
    P[k].M = (uint8_t*)malloc((size_t)Wk * Hk);
    for (int j = 0; j < Hk; ++j)
      for (int i = 0; i < Wk; ++i) {
        int64_t a = (int64_t)(2 * j) * Wf + 2 * i;
        const double* F = P[k - 1].I;
        const uint8_t* FM = P[k - 1].M;
        P[k].I[(int64_t)j * Wk + i] = (((F[a] + F[a + 1]) + F[a + Wf]) + F[a + Wf + 1]) * 0.25;
        P[k].M[(int64_t)j * Wk + i] = (uint8_t)(FM[a] | FM[a + 1] | FM[a + Wf] | FM[a + Wf + 1]);
      }
  }
}

static int est_levels(int W, int H, int levels) {
  int L = levels < 1 ? 1 : levels;
  while (L > 1 && ((W >> (L - 1)) < 8 || (H >> (L - 1)) < 8)) --L;
  return L;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* bilinear sample at (xw, yw) inside [0, W-1] x [0, H-1] (R37: x0 = min(floor(xw), W-2)) */
static double bil(const double* I, int W, int x0, int y0, double fx, double fy) {
  const double* r0 = I + (int64_t)y0 * W + x0;
  const double* r1 = r0 + W;
  return (1.0 - fy) * ((1.0 - fx) * r0[0] + fx * r0[1]) + fy * ((1.0 - fx) * r1[0] + fx * r1[1]);
}

/* central-difference gradient of I at integer (i, j), clamped indices (R37) */
static double gradx(const double* I, int W, int i, int j) {
  int ip = i + 1 < W ? i + 1 : W - 1, im = i - 1 >= 0 ? i - 1 : 0;
  return (I[(int64_t)j * W + ip] - I[(int64_t)j * W + im]) * 0.5;
}
static double grady(const double* I, int W, int H, int i, int j) {
  int jp = j + 1 < H ? j + 1 : H - 1, jm = j - 1 >= 0 ? j - 1 : 0;
  return (I[(int64_t)jp * W + i] - I[(int64_t)jm * W + i]) * 0.5;
}

/* One pixel of frame a at level (W, H): warped position with the parameter vector
 * p = (b_x, s A11, s A12, b_y, s A21, s A22) acting on normalised centred coordinates
 * X = (i - cx) / s, Y = (j - cy) / s (R37).  Returns 1 if the pixel votes. */
static int irls_pixel(const or_grey* A, const or_grey* B, const double* p, double cx, double cy,
                      double s, int i, int j, double* r, int* x0o, int* y0o, double* fxo,
                      double* fyo, double* Xo, double* Yo) {
  int W = A->W, H = A->H;
  if (A->M[(int64_t)j * W + i]) return 0;
  double X = ((double)i - cx) / s, Y = ((double)j - cy) / s;
  double xw = ((p[0] + p[1] * X) + p[2] * Y) + cx;
  double yw = ((p[3] + p[4] * X) + p[5] * Y) + cy;
  if (!(xw >= 0.0 && xw <= (double)(W - 1) && yw >= 0.0 && yw <= (double)(H - 1))) return 0;
  int x0 = (int)floor(xw), y0 = (int)floor(yw);
  if (x0 > W - 2) x0 = W - 2;
  if (y0 > H - 2) y0 = H - 2;
  /* frame b's occlusion: reject if any pixel the sample or its central-difference gradient
   * reads (rows y0-1..y0+2 x cols x0-1..x0+2, clamped) is occluded */
  for (int yy = y0 - 1; yy <= y0 + 2; ++yy)
    for (int xx = x0 - 1; xx <= x0 + 2; ++xx) {
      int cy_ = yy < 0 ? 0 : (yy > H - 1 ? H - 1 : yy), cx_ = xx < 0 ? 0 : (xx > W - 1 ? W - 1 : xx);
      if (B->M[(int64_t)cy_ * W + cx_]) return 0;
    }
  double fx = xw - (double)x0, fy = yw - (double)y0;
  *r = bil(B->I, W, x0, y0, fx, fy) - A->I[(int64_t)j * W + i];
  *x0o = x0; *y0o = y0; *fxo = fx; *fyo = fy; *Xo = X; *Yo = Y;
  return 1;
}

/* 6x6 solve, Gaussian elimination with partial pivoting (first maximal |pivot|); 1 = singular */
static int solve6(double M[6][7], double* x) {
  double md = 0.0;
  for (int k = 0; k < 6; ++k)
    if (fabs(M[k][k]) > md) md = fabs(M[k][k]);
  for (int k = 0; k < 6; ++k) {
    int pr = k;
    for (int r = k + 1; r < 6; ++r)
      if (fabs(M[r][k]) > fabs(M[pr][k])) pr = r;
    if (pr != k)
      for (int c = 0; c < 7; ++c) {
        double tmp = M[k][c]; M[k][c] = M[pr][c]; M[pr][c] = tmp;
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

/* R38: one level of IRLS.  Iteration: (1) residuals r of the voting pixels; n < 12 -> degenerate;
 * (2) sigma = 1.4826 * lower median of |r| (rank floor((n-1)/2)), floored at 1e-6; c = 4.6851
 * sigma; (3) Tukey weights w = (1 - (r/c)^2)^2 for |r| < c, else 0; normal equations of the
 * linearised residual r + J.dp with J = (gx, gx X, gx Y, gy, gy X, gy Y), gx, gy the bilinearly
 * interpolated central-difference gradient of frame b at the warped position, summed exactly as
 * int64 of llrint(term * 2^16); (4) solve (sum w J J^T) dp = -(sum w J r); p += dp; stop when
 * |dp|_2 < tol or after max_iter iterations. */
static int irls_level(const or_grey* A, const or_grey* B, double* p, int max_iter, double tol,
                      int* iters) {
  int W = A->W, H = A->H;
  double cx = (double)(W - 1) * 0.5, cy = (double)(H - 1) * 0.5;
  double s = (double)(W > H ? W : H) * 0.5;
  double* ar = (double*)malloc(sizeof(double) * W * H);
  int status = 0;
  for (int it = 0; it < max_iter; ++it) {
    int64_t n = 0;
    for (int j = 0; j < H; ++j)
      for (int i = 0; i < W; ++i) {
        double r, fx, fy, X, Y;
        int x0, y0;
        if (irls_pixel(A, B, p, cx, cy, s, i, j, &r, &x0, &y0, &fx, &fy, &X, &Y)) ar[n++] = fabs(r);
      }
    if (n < 12) { status = 1; break; }
    qsort(ar, (size_t)n, sizeof(double), cmp_double);
    double sigma = 1.4826 * ar[(n - 1) / 2];
    if (sigma < 1e-6) sigma = 1e-6;
    double c = 4.6851 * sigma;
    int64_t S[6][6] = {{0}}, R[6] = {0};
    for (int j = 0; j < H; ++j)
      for (int i = 0; i < W; ++i) {
        double r, fx, fy, X, Y;
        int x0, y0;
        if (!irls_pixel(A, B, p, cx, cy, s, i, j, &r, &x0, &y0, &fx, &fy, &X, &Y)) continue;
        double u = r / c;
        if (!(fabs(u) < 1.0)) continue;
        double q = 1.0 - u * u;
        double w = q * q;
        double g00 = gradx(B->I, W, x0, y0), g10 = gradx(B->I, W, x0 + 1, y0);
        double g01 = gradx(B->I, W, x0, y0 + 1), g11 = gradx(B->I, W, x0 + 1, y0 + 1);
        double gx = (1.0 - fy) * ((1.0 - fx) * g00 + fx * g10) + fy * ((1.0 - fx) * g01 + fx * g11);
        g00 = grady(B->I, W, H, x0, y0); g10 = grady(B->I, W, H, x0 + 1, y0);
        g01 = grady(B->I, W, H, x0, y0 + 1); g11 = grady(B->I, W, H, x0 + 1, y0 + 1);
        double gy = (1.0 - fy) * ((1.0 - fx) * g00 + fx * g10) + fy * ((1.0 - fx) * g01 + fx * g11);
        double J[6] = {gx, gx * X, gx * Y, gy, gy * X, gy * Y};
        for (int a = 0; a < 6; ++a) {
          double wa = w * J[a];
          for (int b = a; b < 6; ++b) S[a][b] += llrint(wa * J[b] * 65536.0);
          R[a] += llrint(wa * r * 65536.0);
        }
      }
    double M[6][7], dp[6];
    for (int a = 0; a < 6; ++a) {
      for (int b = 0; b < 6; ++b) M[a][b] = (double)(a <= b ? S[a][b] : S[b][a]) / 65536.0;
      M[a][6] = -((double)R[a] / 65536.0);
    }
    ++*iters;
    if (solve6(M, dp)) { status = 1; break; }
    double nrm = 0.0;
    for (int a = 0; a < 6; ++a) {
      p[a] = p[a] + dp[a];
      nrm = nrm + dp[a] * dp[a];
    }
    if (sqrt(nrm) < tol) break;
  }
  free(ar);
  return status;
}

/* parameter vector of level k (coarse) -> level k-1 (fine): centred pixel coordinates satisfy
 * X_fine = 2 X_coarse + d with d = 2 c_coarse + 0.5 - c_fine per axis; (A, b) -> (A, 2b + (I-A)d) */
static void level_up(double* p, int Wc, int Hc, int Wf, int Hf) {
  double sc = (double)(Wc > Hc ? Wc : Hc) * 0.5, sf = (double)(Wf > Hf ? Wf : Hf) * 0.5;
  double a11 = p[1] / sc, a12 = p[2] / sc, a21 = p[4] / sc, a22 = p[5] / sc;
  double dx = ((double)(Wc - 1) + 0.5) - (double)(Wf - 1) * 0.5;
  double dy = ((double)(Hc - 1) + 0.5) - (double)(Hf - 1) * 0.5;
  double bx = 2.0 * p[0] + ((dx - a11 * dx) - a12 * dy);
  double by = 2.0 * p[3] + ((dy - a21 * dx) - a22 * dy);
  p[0] = bx; p[1] = a11 * sf; p[2] = a12 * sf;
  p[3] = by; p[4] = a21 * sf; p[5] = a22 * sf;
}

int or_affine_estimate(const uint8_t* rgb_a, const uint8_t* rgb_b, const uint8_t* occ_a,
                       const uint8_t* occ_b, int W, int H, int levels, int max_iter, double tol,
                       double* theta, int* iters_out) {
  int L = est_levels(W, H, levels);
  or_grey PA[8], PB[8];
  grey_pyr(rgb_a, occ_a, W, H, L, PA);
  grey_pyr(rgb_b, occ_b, W, H, L, PB);
  double s = (double)(PA[L - 1].W > PA[L - 1].H ? PA[L - 1].W : PA[L - 1].H) * 0.5;
  double p[6] = {0.0, s, 0.0, 0.0, 0.0, s};
  int status = 0, iters = 0;
  for (int k = L - 1; k >= 0; --k) {
    if (k < L - 1) level_up(p, PA[k + 1].W, PA[k + 1].H, PA[k].W, PA[k].H);
    status = irls_level(&PA[k], &PB[k], p, max_iter, tol, &iters);
    if (status) break;
  }
  if (status) {
    theta[0] = 0.0; theta[1] = 1.0; theta[2] = 0.0; theta[3] = 0.0; theta[4] = 0.0; theta[5] = 1.0;
  } else {
    /* centred normalised -> spec form: x' = A (x - c) + b + c */
    double s0 = (double)(W > H ? W : H) * 0.5, cx = (double)(W - 1) * 0.5, cy = (double)(H - 1) * 0.5;
    double a11 = p[1] / s0, a12 = p[2] / s0, a21 = p[4] / s0, a22 = p[5] / s0;
    theta[0] = (p[0] + cx) - (a11 * cx + a12 * cy);
    theta[1] = a11; theta[2] = a12;
    theta[3] = (p[3] + cy) - (a21 * cx + a22 * cy);
    theta[4] = a21; theta[5] = a22;
  }
  for (int k = 0; k < L; ++k) { free(PA[k].I); free(PA[k].M); free(PB[k].I); free(PB[k].M); }
  if (iters_out) *iters_out = iters;
  return status;
}

/* R39: 0-based reference m = max(floor(T/2) - 1, 0) (the paper's 1-based N_m = floor(N_f/2));
 * theta_{m,m} = identity; n < m: theta_{n,m} = theta_{n+1,m} o theta_{n,n+1};
 * n > m: theta_{n,m} = theta_{n-1,m} o theta_{n-1,n}^{-1} (Alg. 2, the n > N_m product
 * read as theta^{-1}_{N_m,N_m+1} o ... o theta^{-1}_{n-1,n}). */
int or_affine_chain(const double* pairs, int T, double* fwd, double* inv) {
  int m = T / 2 - 1;
  if (m < 0) m = 0;
  double id[6] = {0.0, 1.0, 0.0, 0.0, 0.0, 1.0};
  for (int i = 0; i < 6; ++i) fwd[6 * m + i] = id[i];
  for (int n = m - 1; n >= 0; --n) or_affine_compose(fwd + 6 * (n + 1), pairs + 6 * n, fwd + 6 * n);
  for (int n = m + 1; n < T; ++n) {
    double pi[6];
    if (or_affine_invert(pairs + 6 * (n - 1), pi)) return 1;
    or_affine_compose(fwd + 6 * (n - 1), pi, fwd + 6 * n);
  }
  for (int n = 0; n < T; ++n)
    if (or_affine_invert(fwd + 6 * n, inv + 6 * n)) return 1;
  return 0;
}

/* R40: clamp-to-edge bilinear sample of an RGB frame at (xs, ys): coordinates clamped to
 * [0, W-1] x [0, H-1], x0 = min(floor, W-2), value rounded half up to u8.  Also reports the
 * footprint pixels with nonzero weight (bit 0: (x0,y0), 1: (x0+1,y0), 2: (x0,y0+1), 3: both). */
static void sample_rgb(const uint8_t* F, int W, int H, double xs, double ys, uint8_t* out, int* x0o,
                       int* y0o, int* fpo) {
  double xc = xs >= 0.0 ? (xs <= (double)(W - 1) ? xs : (double)(W - 1)) : 0.0;
  double yc = ys >= 0.0 ? (ys <= (double)(H - 1) ? ys : (double)(H - 1)) : 0.0;
  int x0 = (int)floor(xc), y0 = (int)floor(yc);
  if (x0 > W - 2) x0 = W - 2;
  if (y0 > H - 2) y0 = H - 2;
  double fx = xc - (double)x0, fy = yc - (double)y0;
  const uint8_t* r0 = F + 3 * ((int64_t)y0 * W + x0);
  const uint8_t* r1 = r0 + 3 * (int64_t)W;
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
  *x0o = x0; *y0o = y0; *fpo = fp;
}

void or_align_warp(const uint8_t* rgb, const uint8_t* occ, int W, int H, int T, const double* inv,
                   uint8_t* rgb_out, uint8_t* mask_out) {
#pragma omp parallel for
  for (int t = 0; t < T; ++t) {
    const double* q = inv + 6 * t;
    const uint8_t* F = rgb + 3 * (int64_t)t * W * H;
    const uint8_t* M = occ + (int64_t)t * W * H;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        double xs = (q[0] + q[1] * (double)x) + q[2] * (double)y;
        double ys = (q[3] + q[4] * (double)x) + q[5] * (double)y;
        int64_t o = ((int64_t)t * H + y) * W + x;
        int x0, y0, fp;
        sample_rgb(F, W, H, xs, ys, rgb_out + 3 * o, &x0, &y0, &fp);
        int invalid = !(xs >= 0.0 && xs <= (double)(W - 1) && ys >= 0.0 && ys <= (double)(H - 1));
        uint8_t m = 0;
        if (invalid) {
          m = 2;
        } else {
          int64_t f = (int64_t)y0 * W + x0;
          if (((fp & 1) && M[f]) || ((fp & 2) && M[f + 1]) || ((fp & 4) && M[f + W]) ||
              ((fp & 8) && M[f + W + 1]))
            m = 1;
        }
        mask_out[o] = m;
      }
  }
}

void or_unwarp(const uint8_t* rgb_aligned, const uint8_t* rgb_orig, const uint8_t* occ_orig, int W,
               int H, int T, const double* fwd, uint8_t* out) {
#pragma omp parallel for
  for (int t = 0; t < T; ++t) {
    const double* q = fwd + 6 * t;
    const uint8_t* F = rgb_aligned + 3 * (int64_t)t * W * H;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        int64_t o = ((int64_t)t * H + y) * W + x;
        if (!occ_orig[o]) {
          out[3 * o] = rgb_orig[3 * o]; out[3 * o + 1] = rgb_orig[3 * o + 1];
          out[3 * o + 2] = rgb_orig[3 * o + 2];
          continue;
        }
        double xs = (q[0] + q[1] * (double)x) + q[2] * (double)y;
        double ys = (q[3] + q[4] * (double)x) + q[5] * (double)y;
        int x0, y0, fp;
        sample_rgb(F, W, H, xs, ys, out + 3 * o, &x0, &y0, &fp);
      }
  }
}
