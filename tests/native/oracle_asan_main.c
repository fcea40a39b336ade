/* Test-only driver: the oracle's whole Alg. 4 (or_inpaint) plus the affine realignment chain,
 * built together with oracle/oracle.c under -fsanitize=address,undefined (tests/test_oracle_asan.py).
 * argv: W H T levels pm_iters fixed_outer rgb.u8 mask.u8 out.u8 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

int main(int argc, char** argv) {
  if (argc != 10) return 2;
  int W = atoi(argv[1]), H = atoi(argv[2]), T = atoi(argv[3]);
  size_t N = (size_t)W * H * T;
  uint8_t* rgb = (uint8_t*)malloc(3 * N);
  uint8_t* occ = (uint8_t*)malloc(N);
  uint8_t* out = (uint8_t*)malloc(3 * N);
  FILE* f = fopen(argv[7], "rb");
  if (!f || fread(rgb, 1, 3 * N, f) != 3 * N) return 3;
  fclose(f);
  f = fopen(argv[8], "rb");
  if (!f || fread(occ, 1, N, f) != N) return 3;
  fclose(f);
  or_params prm;
  memset(&prm, 0, sizeof(prm));
  prm.levels = atoi(argv[4]);
  prm.pm_iters = atoi(argv[5]);
  prm.fixed_outer = atoi(argv[6]);
  prm.max_outer = 20;
  prm.lambda = 50;
  prm.tex_half = -1;
  prm.n_steps = 4;
  prm.steps[0] = 8; prm.steps[1] = 4; prm.steps[2] = 2; prm.steps[3] = 1;
  prm.seed = 1;
  prm.rho = 0.5;
  or_stats st;
  int rc = or_inpaint(rgb, occ, W, H, T, &prm, out, &st);
  if (rc) return 10 + rc;
  /* realignment path: pairwise estimates, chain, warp */
  double* pairs = (double*)calloc(6 * (size_t)(T > 1 ? T - 1 : 1), sizeof(double));
  double* fwd = (double*)calloc(6 * (size_t)T, sizeof(double));
  double* inv = (double*)calloc(6 * (size_t)T, sizeof(double));
  for (int t = 0; t + 1 < T; ++t)
    or_affine_estimate(rgb + 3 * (size_t)W * H * t, rgb + 3 * (size_t)W * H * (t + 1), occ + (size_t)W * H * t,
                       occ + (size_t)W * H * (t + 1), W, H, 3, 20, 1e-4, pairs + 6 * t, NULL);
  or_affine_chain(pairs, T, fwd, inv);
  uint8_t* arg = (uint8_t*)malloc(3 * N);
  uint8_t* am = (uint8_t*)malloc(N);
  or_align_warp(rgb, occ, W, H, T, inv, arg, am);
  f = fopen(argv[9], "wb");
  if (!f || fwrite(out, 1, 3 * N, f) != 3 * N) return 4;
  fclose(f);
  printf("ok outer %d patch-updates %lld\n", st.outer_iters[0], (long long)st.patch_updates[0]);
  free(rgb); free(occ); free(out); free(pairs); free(fwd); free(inv); free(arg); free(am);
  return 0;
}
