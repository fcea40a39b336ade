/* vinp.h — C ABI of the B200 (sm_100a) video-inpainting hot path.
 *
 * Paper: A. Newson, A. Almansa, M. Fradet, Y. Gousseau, P. Perez, "Video inpainting of complex
 * scenes", arXiv 1503.05528.  "P:n" = line n of the paper source; "R<k>" = reading k
 * in DESIGN.md §2 (where the paper is silent or garbled).  Every call below names the passage
 * that defines its operation.
 *
 * Conventions (all calls)
 *  - Buffers are DEVICE pointers owned by the caller (allocated as torch tensors by the Python
 *    binding).  The library never allocates device memory; scratch comes from caller-provided
 *    workspaces whose size is returned by the *_ws_bytes queries.
 *  - `stream` is a cudaStream_t passed as void*.  Calls enqueue work and return without
 *    synchronising, except where a call says it returns host-visible counts.
 *  - Return value: VINP_OK or an error code.  Argument errors are detected synchronously;
 *    device faults surface as VINP_E_CUDA on this or a later call.  vinp_last_error() gives a
 *    thread-local message valid until the next call on that thread.  No C++ exception crosses
 *    the ABI.
 *  - Volumes are t-major: linear index p = (t*H + y)*W + x; this order is also the
 *    lexicographic order of every tie-break (R28).
 *  - Patches are 5x5x5; lambda must lie in [0, 126] so that D fits in 32 bits.
 *
 * Data layout in HBM (one vinp_level per pyramid level, level 1 = finest)
 *  - vox   u64 [T][H][W]: bits 0-7 R, 8-15 G, 16-23 B (working copy u), bits 32-39 T_x,
 *          40-47 T_y in half-grey-level units (T_q = round(2T), Eq. 8, R24); rest 0.
 *  - flags u8  [T][H][W]: bit0 = p in H (occlusion), bit1 = p in D~ (valid source
 *          centre), bit2 = p in H~ (target), bit3 = p in X (invalid: outside
 *          the realigned field of view, NEXT #1 only, R40).
 *  - layer u8  [T][H][W]: onion layer = L_inf distance to D (Alg. 3, R22); coarsest level only,
 *          else NULL.
 *  - slot  i32 [T][H][W]: voxel -> index in `targets`, or -1.
 *  - targets / holes / sources: sorted i32 lists of H~, H and D~.
 *  - NNF (shift map phi) over target slots: e[s] = (D << 32) | q with q = p + phi(p)
 *    the source linear index and D the integer patch distance below; n[s] = |N_p cap Omega cap K|.
 *
 * Integer patch distance (Eq. 9, partial form Eq. 12; R23-R24):
 *    D(p,q) = sum_{r in N_p cap Omega cap K} 4 ||u(r) - u(r-p+q)||^2 + lambda ||T_q(r) - T_q(r-p+q)||^2
 *    d^2(p,q) = D / (4n).
 *  K ("known") is Omega when kb < 0, else {r : layer(r) < kb} (onion peel, Alg. 3).
 *  `only_layer` >= 0 restricts a pass to targets p with layer(p) == only_layer (others are
 *  copied from `in` to `out` unchanged).
 */
#ifndef VINP_H
#define VINP_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VINP_OK = 0,
  VINP_E_INVALID = 1,     /* null pointer, bad shape or range (synchronous) */
  VINP_E_NO_SOURCE = 2,   /* D~ empty at a level: nothing to inpaint from */
  VINP_E_CUDA = 3,        /* launch or runtime error */
  VINP_E_UNSUPPORTED = 4  /* lambda outside [0,126], dims too large, ... */
} vinp_status;

enum { VINP_WEIGHTED = 0, VINP_UNWEIGHTED = 1, VINP_BEST_PATCH = 2 };

typedef struct {
  int32_t W, H, T;   /* dims of this level: W_l = ceil(W/2^(l-1)), T never subsampled */
  int32_t level;     /* 1 = finest; enters the Philox counter */
  uint64_t* vox;
  uint8_t* flags;
  uint8_t* layer;    /* or NULL */
  int32_t* slot;
  int32_t* targets; int32_t n_targets;
  int32_t* holes;   int32_t n_holes;
  int32_t* sources; int32_t n_sources;
  uint16_t* psum;    /* [T][H][W][8] patch sums for the random-search lower bound (R42), or NULL:
                        see vinp_patch_sums */
  uint32_t* active;  /* workspace of vinp_active_ws_bytes(lv) bytes, zeroed once by the caller, or
                        NULL: see vinp_propagate */
} vinp_level;

/* Other ranks' copies of one NNF buffer (NEXT #4 second stage, multi-GPU "fused" exchange): every
 * entry a pass writes into the buffer is also stored, from the same kernel, into each peer copy
 * (peer-mapped device pointers, e.g. torch symmetric memory; P2P stores over NVLink) and/or through
 * an NVLS multicast address of the e array (multimem.st: one store reaches every GPU's copy).  The
 * caller orders passes across ranks (a barrier after each pass); the library never waits. */
#define VINP_MAX_PEERS 7
typedef struct {
  int32_t n_peers;                    /* 0..VINP_MAX_PEERS */
  uint64_t* e[VINP_MAX_PEERS];        /* peer copies of e */
  uint8_t* n[VINP_MAX_PEERS];         /* peer copies of n (written by evaluate), or NULL */
  uint8_t* stamp[VINP_MAX_PEERS];     /* peer copies of stamp, or NULL */
  uint64_t* mc_e;                     /* NVLS multicast address of e, or NULL (then e[] is used) */
} vinp_mirror;

typedef struct {
  uint64_t* e;      /* [n_targets] (D << 32) | source index */
  uint8_t* n;       /* [n_targets] patch voxel count; may be shared by ping-pong buffers */
  uint8_t* stamp;   /* [n_targets] or NULL: index of the pass of the current ANN search that last
                       changed e[s] (0 = unchanged since its evaluate); one array per ping-pong
                       buffer.  Enables the exact stale-candidate skip of vinp_propagate (R41). */
  const vinp_mirror* mirror;  /* NULL, or where the entries written into this buffer also go */
} vinp_nnf;

typedef struct {
  int32_t lambda;    /* texture weight, 50 */
  int32_t tex_half;  /* half-width h of the texture window nu (R15); -1 = max(1, 2^(L-2)) */
  uint64_t seed;     /* Philox key */
  double rho;        /* random-search window reduction, 0.5 */
  int32_t rmax;      /* random-search radius; -1 = max(W_l, H_l, T) (R7) */
} vinp_params;

const char* vinp_last_error(void);
int vinp_version(void);
/* Pyramid dimensions: dims_out[3l .. 3l+2] = (W_l, H_l, T) for l = 1..L, with
 * W_l = ceil(W_{l-1} / 2), H_l likewise and T never subsampled.  Host-only; VINP_E_INVALID for
 * non-positive sizes or L outside [1, 16], VINP_E_UNSUPPORTED if W*H*T >= 2^31. */
vinp_status vinp_level_dims(int W, int H, int T, int L, int32_t* dims_out);

/* Number of kernels this library has launched since it was loaded (evidence counter). */
uint64_t vinp_launch_count(void);

/* ---- a1: video + occlusion pyramid (Alg. 4; spatial only P:878-882; R17/R18) ----
 * rgb: u8 [T][H][W][3] and mask: u8 [T][H][W], device, level-1 dims.  Mask codes: 0 known,
 * 2 = invalid X (a realigned pixel whose source lies outside its frame, R40; a known voxel that
 * no source patch may contain), any other nonzero = occluded (H).
 * Writes vox colour bytes and flags bits 0 and 3 of levels 1..L (lv[0..L-1]); texture bytes are
 * zeroed.  Coarse value = round-half-up of the binomial (1,4,6,4,1)^2 mean over unoccluded fine
 * voxels (reflect-101 borders), 0 if none; coarse occluded (invalid) iff any of its 2x2 fine
 * voxels is. */
vinp_status vinp_build_pyramid(const uint8_t* rgb, const uint8_t* mask, vinp_level* lv, int L,
                               void* stream);

/* ---- a3: texture features + texture pyramid (Eq. 8; Eq. 10; R14-R16) ----
 * Computes T on level 1 from its colour and occlusion (masked central differences of the
 * x1000 Rec.601 luma, mean over the (2h+1)^2 window) and writes T^l(x,y,t) = T(2^(l-1)x,
 * 2^(l-1)y, t) into the texture bytes of every level.  ws: vinp_texture_ws_bytes(lv[0]). */
size_t vinp_texture_ws_bytes(const vinp_level* lv1);
vinp_status vinp_texture_features(const vinp_params* prm, vinp_level* lv, int L, void* ws,
                                  size_t ws_bytes, void* stream);

/* ---- a2: source/target sets ----
 * vinp_build_sets: flags bit1 (D~: N_p inside Omega and disjoint from H and X) and bit2 (H~)
 * from bits 0 and 3 for levels 1..L, and returns the
 * list sizes in counts_out[3l+0..2] = |H~|, |H|, |D~| (host memory; this call synchronises).
 * vinp_build_lists: fills targets/holes/sources (ascending) and slot for levels 1..L into
 * caller buffers sized from those counts; sets lv[l].n_*.  ws: vinp_sets_ws_bytes. */
size_t vinp_sets_ws_bytes(const vinp_level* lv1);
vinp_status vinp_build_sets(vinp_level* lv, int L, int32_t* counts_out, void* ws, size_t ws_bytes,
                            void* stream);
vinp_status vinp_build_lists(vinp_level* lv, int L, void* ws, size_t ws_bytes, void* stream);

/* ---- Alg. 3 onion layers: layer(p) = L_inf distance from p to D, out-of-bounds occluded (R22).
 * Writes lv->layer; *n_layers_out = max layer (host; synchronises).  ws: >= 16 device bytes. */
vinp_status vinp_layers(vinp_level* lv, int32_t* n_layers_out, void* ws, void* stream);

/* ---- a5: NNF initialisation ----
 * Random (Alg. 4; R8): q = sources[(U0 |D~|) >> 32], U0 = Philox(p, 0,
 * (level<<24)|(1<<16), outer_code).  Upsample (Alg. 4; R21): fine shift =
 * (2dx, 2dy, dt) of the coarse shift at (x/2, y/2, t); invalid results are re-drawn with stream 3.
 * Evaluate: (D, n) of the current shift on the current u and K.  All act on target slots
 * [b, e).  D of init/upsample is left 0 until evaluate. */
vinp_status vinp_nnf_init_random(const vinp_level* lv, vinp_nnf* nnf, const vinp_params* prm,
                                 uint32_t outer_code, int32_t b, int32_t e, void* stream);
vinp_status vinp_nnf_upsample(const vinp_level* coarse, const vinp_nnf* cn, const vinp_level* fine,
                              vinp_nnf* fn, const vinp_params* prm, int32_t b, int32_t e,
                              void* stream);
/* Evaluate also sets stamp[s] = 0 for every slot of [b, e) (filtered-out slots included) when
 * nnf->stamp is given: it starts the pass numbering of an ANN search. */
vinp_status vinp_nnf_evaluate(const vinp_level* lv, vinp_nnf* nnf, const vinp_params* prm, int kb,
                              int only_layer, int32_t b, int32_t e, unsigned long long* counter,
                              void* stream);

/* ---- a6: propagation, one Jacobi jump pass (Alg. 1; R2, R5, R6, R25) ----
 * Candidates in rank order: 0 = in(p); 1..3 = in(p + sign*step*e_x / e_y / e_t) for neighbours in
 * Omega and H~ (sign = 0: 1..6 = the -step then the +step neighbours).  A candidate is evaluated iff q = p + v is in Omega and D~ and v differs from the
 * incumbent and from every earlier valid candidate; strict improvement wins.  Reads `in`, writes
 * `out` for slots [b, e).  counter (device, may be NULL) += evaluated candidates.
 * Stale skip (R41; only if in->stamp and out->stamp are both given, else both must be NULL):
 * `pass` in [1, 255] is this pass's index in the current ANN search (evaluate = 0) and `since`
 * the index of the previous pass with the same (step, sign) in that search (0 = none).  A
 * candidate whose neighbour r has in->stamp[r] < since proposes the shift it proposed at pass
 * `since`; it was then tested against this target (or equalled its incumbent), whose D has not
 * grown since, so it cannot win (strict improvement) and is not evaluated: the NNF is identical
 * to the unskipped pass.  Such candidates are counted in counter[1] (counter then points to two
 * u64), not in counter[0].  out->stamp[s] = pass if e[s] changed, else in->stamp[s].
 * With lv->active set (passes with since > 0, only_layer < 0 and no mirror), a first kernel copies
 * the entries and stamps of [b, e) to `out` and lists the targets of [b, e) that read an entry
 * changed since `since` (in->stamp must be current for every target those targets read: the whole
 * level, or a slab plus its halo rows); the pass then runs over that list alone: the other targets receive stale proposals
 * only and keep their entry.  The NNF, the stamps and counter[0] are identical; counter[1] is then
 * NOT updated (the stale candidates of unlisted targets are never enumerated). */
vinp_status vinp_propagate(const vinp_level* lv, const vinp_nnf* in, vinp_nnf* out,
                           const vinp_params* prm, int step, int sign, int kb, int only_layer,
                           int32_t b, int32_t e, int pass, int since, unsigned long long* counter,
                           void* stream);

/* ---- patch sums for an exact lower-bound rejection in random search (R42; an early termination
 * that changes no comparison, like R35) ----
 * psum[p] = (S_R, S_G, S_B, S_Tx, S_Ty, 0, 0, 0), u16: the sums of the five channels of vox over
 * the 125 voxels of N_p, defined for voxels whose whole patch lies in Omega (others: 0, never used).
 * For a target p with a full patch and a source q in D~ (whose patch is always full), Cauchy-Schwarz
 * over the 125 voxels gives, with the integer distance D of this header,
 *     125 D(p, q) >= 4 (dS_R^2 + dS_G^2 + dS_B^2) + lambda (dS_Tx^2 + dS_Ty^2),  dS = S(p) - S(q),
 * so a candidate whose right-hand side is >= 125 D_incumbent cannot strictly improve (R25) and is
 * rejected by vinp_random_search (kb < 0 launches) before any patch row is read.  It still counts
 * as a patch-update: results and counts equal those without psum.
 * which = 0: every voxel (once per level, after vinp_texture_features: covers D~, which never
 * changes); which = 1: the targets of slots [b, e) on the current u.  vinp_nnf_evaluate with kb < 0
 * and only_layer < 0 refreshes the targets of its slots itself when lv->psum is set, so a search
 * that starts with evaluate (as every ANN search does) always sees sums of the current u.
 * VINP_E_INVALID if lv->psum is NULL. */
vinp_status vinp_patch_sums(const vinp_level* lv, int which, int32_t b, int32_t e, void* stream);

/* Bytes of the lv->active workspace (list length, a bitmap over the target slots, the list) for
 * lv->n_targets targets; the caller zeroes it once after vinp_build_sets. */
size_t vinp_active_ws_bytes(const vinp_level* lv);

/* ---- a7: random search (Eq. 3, Alg. 1; R1, R3, R7) ----
 * v0 = in(p); for i = 1, 2, ...: R_i = rmax * rho^i (repeated fp64 multiplication) while
 * R_i >= 1; delta_c = (U_c - 2^31) 2^-31 from Philox(p, pm_iter, (level<<24)|(2<<16)|i,
 * outer_code); q_i = p + v0 + floor(R_i delta).  Same validity / duplicate / strict rules.
 * With stamps (as vinp_propagate), out->stamp[s] = pass if e[s] changed, else in->stamp[s].
 * counter (device, may be NULL) += the valid, distinct candidates tested against the incumbent,
 * whether by their full distance, by a partial sum that already exceeds the best (R35) or, with
 * lv->psum, by the patch-sum lower bound (R42, see vinp_patch_sums): the same number in all cases. */
vinp_status vinp_random_search(const vinp_level* lv, const vinp_nnf* in, vinp_nnf* out,
                               const vinp_params* prm, uint32_t outer_code, int pm_iter, int kb,
                               int only_layer, int32_t b, int32_t e, int pass,
                               unsigned long long* counter, void* stream);

/* ---- a8: ANN search (Alg. 1), single GPU: evaluate, then for k = 1..K: for each step
 * s in steps: propagate(s, sign); random_search(k).  sign_policy 0: sign = +1 for odd k, -1 for
 * even k (Alg. 1's alternation, R5); 1: sign = 0 (both directions) on every pass (R6).  Uses `b`
 * as the ping-pong buffer; the result is in `a`.  With stamps on both buffers, passes are numbered
 * 1, 2, ... in schedule order and the R41 stale skip is applied (counter[1], see vinp_propagate);
 * if K * (n_steps + 1) > 255 the search runs without it. */
vinp_status vinp_ann_search(const vinp_level* lv, vinp_nnf* a, vinp_nnf* b, const vinp_params* prm,
                            uint32_t outer_code, int K, const int32_t* steps, int n_steps,
                            int sign_policy, int kb, int only_layer, unsigned long long* counter,
                            void* stream);

/* ---- a9/a10: reconstruction (Eqs. 4-5, Eq. 6, Eq. 11, Eq. 13
 * P:829-832; R10-R13, R20, R26, R27) ----
 * For holes[h], h in [hb, he) (and layer(p) == layer_j if layer_j >= 0): contributors q in
 * N_p cap Omega (with layer(q) < layer_j for an onion layer).  mode VINP_WEIGHTED: sigma^2 = the
 * ceil(0.75 m)-th smallest d^2_q (exact rationals), weights round(exp(-a_q) 2^36) with
 * a_q = D_q n_s / (2 n_q D_s); mean over zero-distance contributors if sigma = 0.
 * VINP_UNWEIGHTED: weights 1.  VINP_BEST_PATCH: copy from argmin d^2_q (ties -> smallest q).
 * Writes out_rgb[h][3], out_tex[h][2] (fp32; texture in half-grey units) and, if commit != 0,
 * the u8 working copy floor(x + 0.5) into vox at p. */
vinp_status vinp_reconstruct(vinp_level* lv, const vinp_nnf* nnf, int mode, int layer_j, int32_t hb,
                             int32_t he, float* out_rgb, float* out_tex, int commit, void* stream);
/* Write floor(x + 0.5) of out_rgb/out_tex for holes [hb, he) (layer_j filter as above) into vox. */
vinp_status vinp_commit(vinp_level* lv, const float* out_rgb, const float* out_tex, int layer_j,
                        int32_t hb, int32_t he, void* stream);

/* ---- a12: onion-peel initialisation (Alg. 3; Eqs. 12-13; R22), coarsest level, after
 * vinp_layers and vinp_nnf_init_random on `a`: for j = 0..n_layers: ANN search (as vinp_ann_search,
 * K iterations, outer code 0x80000000|j) over the targets with layer(p) == j and known set
 * K = {layer < max(j,1)}; then for j >= 1 the weighted reconstruction (Eq. 13) of the holes of
 * layer j, committed to the working copy.  Layer-j index lists are built once in ws
 * (vinp_onion_ws_bytes); synchronises once.  Result NNF in `a`; `b` is scratch. */
size_t vinp_onion_ws_bytes(const vinp_level* lv);
vinp_status vinp_onion_peel(vinp_level* lv, vinp_nnf* a, vinp_nnf* b, const vinp_params* prm, int K,
                            const int32_t* steps, int n_steps, int sign_policy, int n_layers, float* out_rgb,
                            float* out_tex, unsigned long long* counter, void* ws, size_t ws_bytes,
                            void* stream);

/* ---- a11: stopping-rule change (Alg. 4, R19): *out (device int64) += sum_i
 * llrint(|a_i - b_i| 2^20).  e = out / 2^20 / (3|H|). */
vinp_status vinp_change_l1(const float* a, const float* b, int64_t n, int64_t* out, void* stream);
/* The literal P:988 statistic (Config stop_rule = 1): *out += sum_i llrint((a_i - b_i)^2 2^20) (the
 * square of a float difference is exact in fp64); e = sqrt(out / 2^20) / (3|H|).  Same buffers and
 * errors as vinp_change_l1. */
vinp_status vinp_change_l2(const float* a, const float* b, int64_t n, int64_t* out, void* stream);

/* ---- Eq. 1 P:286-289 (diagnostic): *out (device double) = sum_{p in H} D_p / (4 n_p). */
vinp_status vinp_energy(const vinp_level* lv, const vinp_nnf* nnf, double* out, void* stream);

/* ---- a13: exact NN (definition of Matching): argmin over q in D~ of D(p, q), K = Omega,
 * ties -> smallest q; target slots [b, e).  The CUDA-core form needs no workspace:
 * vinp_brute_force_ws_bytes returns 0 and ws may be NULL.  Errors: VINP_E_INVALID (null buffers,
 * bad range), VINP_E_UNSUPPORTED (lambda outside [0,126]), VINP_E_NO_SOURCE (D~ empty), all
 * synchronous. */
size_t vinp_brute_force_ws_bytes(const vinp_level* lv);
vinp_status vinp_brute_force(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm, int32_t b,
                             int32_t e, void* ws, size_t ws_bytes, void* stream);
/* The same exact NN over an explicit device list of n target slots (CUDA cores); every list entry
 * must lie in [0, n_targets).  Same synchronous argument errors as vinp_brute_force (the list's
 * contents live on the device and are not inspected). */
vinp_status vinp_brute_force_list(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm,
                                  const int32_t* list, int32_t n, void* stream);
/* Tensor-core form (north_star: "optional exact brute-force NN mode expressed as a dense
 * contraction"): for targets whose patch lies inside Omega, D(p,q) = E(p) + E(q) - 2(4 X_c + lambda
 * X_t) with X the u8 patch dot products computed by tcgen05.mma kind::i8 (colour K = 384, texture
 * K = 256), minimised exactly in the epilogue (ties -> smallest q); border targets go to the CUDA-core
 * path.  Same result as vinp_brute_force, bit for bit.  Synchronises once (target counts).
 * ws: vinp_brute_force_tc_ws_bytes(lv, b, e) (holds the im2col rows: 640 B per target and source). */
size_t vinp_brute_force_tc_ws_bytes(const vinp_level* lv, int32_t b, int32_t e);
vinp_status vinp_brute_force_tc(const vinp_level* lv, vinp_nnf* out, const vinp_params* prm, int32_t b,
                                int32_t e, void* ws, size_t ws_bytes, void* stream);

/* ---- App. B Monte-Carlo (Table 2; NEXT #3): *hits (device) += number of trials t in
 * [trial0, trial0 + n_trials) in which a random patch V beats the constant patch Z = mu for a random
 * reference W (N i.i.d. N(mu, sigma^2) components; fp64 Box-Muller on Philox, counter (t lo, t hi,
 * 4<<16 | k, 0)).  Probability estimate = hits / n_trials. */
vinp_status vinp_patch_ambiguity(int N, double sigma, uint64_t seed, uint64_t trial0, uint64_t n_trials,
                                 unsigned long long* hits, void* stream);

/* ---- NEXT #1: dominant affine motion and realignment (Alg. 2; S3.4 P:744-758) ----
 * theta = 6 doubles (a1..a6): (x, y) -> (a1 + a2 x + a3 y, a4 + a5 x + a6 y) in full-resolution
 * pixel coordinates (x column, y row).  All buffers device, caller-owned.
 *
 * vinp_affine_estimate: theta[n] (n < T-1) = theta_{n,n+1}, the dominant motion from frame n to
 *   n+1 (I_{n+1}(theta(x)) ~ I_n(x)), by robust IRLS (R36-R38: grey pyramid of `levels` 2x2 box
 *   levels (fewer while the coarsest side would be < 8), Tukey biweight, scale 1.4826 x exact
 *   lower median of |r|, <= max_iter iterations per level or |dp| < tol).  Pixels with mask != 0
 *   are excluded (in frame n as voters; in frame n+1 from every sample/gradient footprint).
 *   status[n] = 0, or 1 = degenerate (fewer than 12 voters or singular normal equations), in
 *   which case theta[n] = identity; iters[n] = IRLS iterations run.  Deterministic and
 *   bit-identical to the oracle (exact fixed-point sums, no FMA contraction).  One 8-CTA cluster per pair.
 *   Only pairs n in [pair_b, pair_e) are estimated (pair_e < 0: up to T-1), so ranks can split the
 *   independent pairs; rows outside the range are not written.
 *   ws: vinp_affine_ws_bytes(W, H, T, levels) (grey pyramids + |r| keys).
 * vinp_affine_chain: fwd[n] = theta_{n,N_m} (frame n -> reference frame N_m = max(T/2 - 1, 0),
 *   0-based, R39) by the products of Alg. 2, inv[n] = fwd[n]^-1; *err (device) = 1 if a map
 *   was singular.  One thread (the chain is sequential by definition).
 * vinp_align_warp: aligned frame n at reference pixel y = frame n sampled bilinearly at inv[n](y)
 *   (clamp-to-edge, rounded half up to u8); mask_out = 2 where inv[n](y) falls outside frame n,
 *   else 1 iff a nonzero-weight footprint pixel is occluded (mask != 0), else 0 (R40).
 * vinp_unwarp: out = rgb_orig where mask_orig == 0; inside the original occlusion, the inpainted
 *   aligned video sampled bilinearly at fwd[n](x) (clamp-to-edge, rounded half up) (R40). */
size_t vinp_affine_ws_bytes(int W, int H, int T, int levels);
vinp_status vinp_affine_estimate(const uint8_t* rgb, const uint8_t* mask, int W, int H, int T, int levels,
                                 int max_iter, double tol, int32_t pair_b, int32_t pair_e, double* theta,
                                 int32_t* status, int32_t* iters, void* ws, size_t ws_bytes, void* stream);
vinp_status vinp_affine_chain(const double* pairs, int T, double* fwd, double* inv, int32_t* err,
                              void* stream);
vinp_status vinp_align_warp(const uint8_t* rgb, const uint8_t* mask, int W, int H, int T, const double* inv,
                            uint8_t* rgb_out, uint8_t* mask_out, void* stream);
vinp_status vinp_unwarp(const uint8_t* rgb_aligned, const uint8_t* rgb_orig, const uint8_t* mask_orig, int W,
                        int H, int T, const double* fwd, uint8_t* out, void* stream);
/* Final video of level 1: out[p] = the RGB bytes of vox[p] (input outside H, inpainted inside). */
vinp_status vinp_output_rgb(const vinp_level* lv1, uint8_t* out, void* stream);

/* ---- test hooks ----
 * vinp_patch_ssd: D and n of pairs (p[i], q[i]) with known set kb (q must be in D~).
 * vinp_philox: out[i][0..3] = Philox4x32-10(ctr[i][0..3], key = seed).
 * vinp_tc_gemm_u8: C[128][128] (s32) = A[128][K] * B[128][K]^T for u8 A, B (K % 32 == 0, K <= 512),
 * one tcgen05.mma kind::i8 tile — pins the tensor-core plumbing used by the exact NN mode. */
vinp_status vinp_patch_ssd(const vinp_level* lv, const int32_t* p, const int32_t* q, int64_t n,
                           const vinp_params* prm, int kb, uint32_t* D, uint8_t* cnt, void* stream);
vinp_status vinp_philox(const uint32_t* ctr, int64_t n, uint64_t seed, uint32_t* out, void* stream);
vinp_status vinp_tc_gemm_u8(const uint8_t* A, const uint8_t* B, int K, int32_t* C, void* stream);

#ifdef __cplusplus
}
#endif
#endif
