/* oracle.h — plain, slow, obviously-correct CPU oracle of the inpainting hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1503_05528_b200/) never links, imports or calls it, and shares no code
 * with it (no common headers, kernels, helpers or constant tables).
 *
 * Paper: Newson et al., "Video inpainting of complex scenes", arXiv 1503.05528.
 * Citations "P:n" are PAPER.md line numbers; "R<k>" are the readings listed in
 * DESIGN.md §2 (the paper's silent/garbled points and the reading adopted).
 *
 * Data model (independent of the GPU layout):
 *   colour   u8  [T][H][W][3]        (u : Omega -> R^3)
 *   texture  u8  [T][H][W][2]        half-grey-level units, T_q = round(2T)  (Eq. 8; R24)
 *   occ      u8  [T][H][W]           1 = in H
 *   src/tgt  u8  [T][H][W]           membership of D~ / H~
 *   NNF      over the sorted target list: dx,dy,dt (int32), D (u32), n (u8)   (phi)
 * Linear index p = (t*H + y)*W + x; t-major order is the lexicographic order (R28).
 *
 * Parity status: every function here is pinned by a `-m "not gpu"` test except
 * where its comment says "parity unpinned".
 */
#ifndef VINP_ORACLE_H
#define VINP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int W, H, T;
  uint8_t* rgb;      /* [N][3] */
  uint8_t* tex;      /* [N][2] */
  uint8_t* occ;      /* [N]    */
  uint8_t* src;      /* [N] D~ */
  uint8_t* tgt;      /* [N] H~ */
  uint8_t* layer;    /* [N] onion layer (coarsest level) or NULL */
  int32_t* slot;     /* [N] voxel -> target slot or -1 */
  int32_t* targets; int32_t n_targets;
  int32_t* holes;   int32_t n_holes;
  int32_t* sources; int32_t n_sources;
} or_level;

typedef struct {
  int32_t *dx, *dy, *dt;
  uint32_t* D;
  uint8_t* n;
} or_nnf;

enum { OR_WEIGHTED = 0, OR_UNWEIGHTED = 1, OR_BEST_PATCH = 2 };

void or_philox4x32_10(const uint32_t ctr[4], uint64_t seed, uint32_t out[4]);

void or_pyramid_down(const uint8_t* rgb, const uint8_t* occ, int W, int H, int T,
                     uint8_t* rgb_c, uint8_t* occ_c);
void or_texture(const uint8_t* rgb, const uint8_t* occ, int W, int H, int T, int h, uint8_t* tex);
void or_texture_decimate(const uint8_t* tex1, int W1, int H1, int T, int level,
                         int Wl, int Hl, uint8_t* texl);
void or_sets(const uint8_t* occ, int W, int H, int T, uint8_t* src, uint8_t* tgt);
int or_layers(const uint8_t* occ, int W, int H, int T, uint8_t* layer);

void or_patch_ssd(const or_level* lv, int32_t p, int32_t q, int lambda, int kb,
                  uint32_t* D, uint32_t* n);

int64_t or_nnf_init_random(const or_level* lv, or_nnf* nnf, uint64_t seed, int level,
                           uint32_t outer_code, int32_t b, int32_t e);
void or_nnf_upsample(const or_level* coarse, const or_nnf* cn, const or_level* fine, or_nnf* fn,
                     uint64_t seed, int level, int32_t b, int32_t e);
int64_t or_nnf_evaluate(const or_level* lv, or_nnf* nnf, int lambda, int kb, int only_layer,
                        int32_t b, int32_t e);
/* prev (may be NULL): the input NNF of the previous pass with the same (step, sign) in the same
 * ANN search; *stale (may be NULL) receives how many of the evaluated candidates equal the shift
 * their neighbour held in prev (R41: a count only, the pass itself is unchanged) */
int64_t or_propagate(const or_level* lv, const or_nnf* in, or_nnf* out, int lambda, int step,
                     int sign, int kb, int only_layer, int32_t b, int32_t e, const or_nnf* prev,
                     int64_t* stale);
int64_t or_random_search(const or_level* lv, const or_nnf* in, or_nnf* out, int lambda,
                         uint64_t seed, double rho, int rmax, int level, uint32_t outer_code,
                         int pm_iter, int kb, int only_layer, int32_t b, int32_t e);
void or_reconstruct(or_level* lv, const or_nnf* nnf, int mode, int layer_j, int32_t hb, int32_t he,
                    float* out_rgb, float* out_tex);
void or_commit(or_level* lv, const float* out_rgb, const float* out_tex, int32_t hb, int32_t he);
int64_t or_change_l1(const float* a, const float* b, int64_t n);
/* literal P:988 variant: sum over hole channels of llrint((a-b)^2 2^20) ((a-b)^2 is exact in fp64) */
int64_t or_change_l2(const float* a, const float* b, int64_t n);
double or_energy(const or_level* lv, const or_nnf* nnf);
int64_t or_brute_force(const or_level* lv, or_nnf* out, int lambda, int32_t b, int32_t e);

/* App. B, Table 2 (NEXT #3): probability that a random patch V is closer (SSD) to a
 * random reference patch W than the constant patch Z = mu, components i.i.d. N(mu, sigma^2).
 * Exact value P_N = E[Q(sqrt(chi2_N) / 2)] (1-D integral, independent of sigma), and the paper's
 * direct simulation on the CPU (fp64 Box-Muller on this oracle's Philox; counter (trial lo,
 * trial hi, 4 << 16 | component pair, 0)). */
double or_ambiguity_exact(int N);
int64_t or_ambiguity_mc(int N, double sigma, uint64_t seed, uint64_t trial0, uint64_t n_trials);

/* NEXT #2: Alg. 1 as printed — in-place lexicographic scans: even k forward with
 * the -1 neighbours, odd k reverse with the +1 neighbours (reusing entries already
 * updated in the same scan), then an in-place random search over the targets in lexicographic
 * order (Eq. 3 with the R3 inner loop, centred on the current phi(p)).  Same validity,
 * de-duplication and strict-improvement rules as the Jacobi passes.  Starts with an evaluate.
 * Single-threaded by definition.  Returns the number of evaluated candidates. */
int64_t or_ann_search_sequential(const or_level* lv, or_nnf* nnf, int lambda, uint64_t seed,
                                 double rho, int rmax, int level, uint32_t outer_code, int K);

/* a2 with the realignment's invalid set X (R40): D~ = {p : N_p inside Omega, N_p  disjoint from
 * H and X}; H~ as or_sets.  inv may be NULL (= or_sets). */
void or_sets_x(const uint8_t* occ, const uint8_t* inv, int W, int H, int T, uint8_t* src,
               uint8_t* tgt);
/* any-of-2x2 decimation of a 0/1 mask (R18; used for X) */
void or_mask_down(const uint8_t* m, int W, int H, int T, uint8_t* mc);

/* ---- NEXT #1: dominant affine motion and realignment (Alg. 2; S3.4 P:744-758) ----
 * theta = (a1..a6): (x, y) -> (a1 + a2 x + a3 y, a4 + a5 x + a6 y), full-resolution pixel
 * coordinates (x = column, y = row), theta_{n,n+1} maps frame n to frame n+1:
 * I_{n+1}(theta(x)) ~ I_n(x).  Readings R36-R40. */
void or_affine_compose(const double* t2, const double* t1, double* out); /* t2 o t1 */
int or_affine_invert(const double* t, double* out);                     /* 0 ok, 1 singular */
/* Robust IRLS estimate between two frames (R36-R38); occ_a excludes pixels of frame a, occ_b
 * the footprints in frame b (NULL = none).  Returns 0, or 1 = degenerate (theta = identity).
 * iters_out (may be NULL) = total IRLS iterations over all levels. */
int or_affine_estimate(const uint8_t* rgb_a, const uint8_t* rgb_b, const uint8_t* occ_a,
                       const uint8_t* occ_b, int W, int H, int levels, int max_iter, double tol,
                       double* theta, int* iters_out);
/* theta_{n,Nm} for every frame (Alg. 2 second loop, R39) and its inverse; 0 ok, 1 singular */
int or_affine_chain(const double* pairs, int T, double* fwd, double* inv);
/* aligned frame n = u_n sampled bilinearly at inv[n](y) (R40); mask_out: 0, 1 = occluded (any
 * nonzero-weight footprint pixel occluded), 2 = invalid (source outside frame n) */
void or_align_warp(const uint8_t* rgb, const uint8_t* occ, int W, int H, int T, const double* inv,
                   uint8_t* rgb_out, uint8_t* mask_out);
/* inverse warp of the inpainted aligned video, pasted into the original occluded pixels only */
void or_unwarp(const uint8_t* rgb_aligned, const uint8_t* rgb_orig, const uint8_t* occ_orig, int W,
               int H, int T, const double* fwd, uint8_t* out);

/* Whole Alg. 4 on host buffers; occ codes 0 known, 1 occluded (H), 2 invalid (X, R40, only
 * after realignment).  Returns 0 on success. */
typedef struct {
  int levels, pm_iters, fixed_outer, max_outer, lambda, tex_half, n_steps, sign_policy;
  int steps[8];
  uint64_t seed;
  double rho;
  int stop_rule; /* 0: R19 e = ||u_H - v_H||_1 / (3|H|); 1: literal P:988 ||u_H - v_H||_2 / (3|H|) */
} or_params;
typedef struct {
  int outer_iters[16];
  int64_t patch_updates[16];
  int onion_layers;
  /* diagnostics for the pins: the change statistic of every outer iteration (fixed point 2^20,
   * or_change_l1 / or_change_l2 by stop_rule; first 32 iterations), |H| per level, and how many
   * hole voxels the onion peel committed (each exactly once) */
  int64_t change_fixed[16][32];
  int64_t n_holes[16];
  int64_t onion_commits;
  /* per level: evaluated propagation candidates that were stale (R41), included in patch_updates */
  int64_t stale[16];
} or_stats;
/* R19 / P:930-939 stopping decision after outer iteration k (1-based) of a level with n_holes
 * hole voxels: 1 = stop.  stop_rule 0: e_fixed = sum llrint(|a-b| 2^20), stop iff
 * e_fixed / 2^20 / (3 n_holes) <= 0.1; stop_rule 1: e_fixed = sum llrint((a-b)^2 2^20), stop iff
 * sqrt(e_fixed / 2^20) / (3 n_holes) <= 0.1.  Always stop at k >= max_outer. */
int or_stop(int64_t e_fixed, int64_t n_holes, int k, int max_outer, int stop_rule);
int or_inpaint(const uint8_t* rgb, const uint8_t* occ, int W, int H, int T, const or_params* prm,
               uint8_t* out_rgb, or_stats* st);

#ifdef __cplusplus
}
#endif
#endif
