/* c_pipeline.c — Alg. 4 at one pyramid level with a fixed number of outer iterations, driven
 * through the raw C ABI of libvinp (include/vinp.h) with no Python or torch: device buffers from
 * cudaMalloc, the same call sequence as paper_1503_05528_b200/driver.py.
 *
 *   onion peel (Alg. 3) -> repeat outer { ANN search (Alg. 1); weighted reconstruction (Eqs. 4-5) }
 *   -> best-patch reconstruction (Eq. 6) -> output video
 *
 * usage: c_pipeline W H T K OUTER in_rgb in_mask out_rgb
 *   in_rgb: T*H*W*3 u8, in_mask: T*H*W u8 (nonzero = occluded), raw files; out_rgb likewise.
 * build: gcc -O2 -std=c11 -I include -I /usr/local/cuda/include examples/c_pipeline.c \
 *          -L paper_1503_05528_b200 -lvinp -L /usr/local/cuda/lib64 -lcudart \
 *          -Wl,-rpath,$PWD/paper_1503_05528_b200 -o c_pipeline                            */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "vinp.h"

#define CK(x)                                                           \
  do {                                                                  \
    vinp_status s_ = (x);                                               \
    if (s_ != VINP_OK) {                                                \
      fprintf(stderr, "%s failed (%d): %s\n", #x, s_, vinp_last_error()); \
      return 1;                                                         \
    }                                                                   \
  } while (0)

static void* dalloc(size_t n) {
  void* p = NULL;
  if (n == 0) n = 16;
  if (cudaMalloc(&p, n) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc(%zu) failed\n", n);
    exit(1);
  }
  cudaMemset(p, 0, n);
  return p;
}

static int read_file(const char* path, void* buf, size_t n) {
  FILE* f = fopen(path, "rb");
  if (!f) return 1;
  size_t r = fread(buf, 1, n, f);
  fclose(f);
  return r != n;
}

int main(int argc, char** argv) {
  if (argc != 9) {
    fprintf(stderr, "usage: %s W H T K OUTER in_rgb in_mask out_rgb\n", argv[0]);
    return 2;
  }
  const int W = atoi(argv[1]), H = atoi(argv[2]), T = atoi(argv[3]), K = atoi(argv[4]);
  const int outer = atoi(argv[5]);
  const size_t N = (size_t)W * H * T;
  uint8_t* rgb = (uint8_t*)malloc(3 * N);
  uint8_t* mask = (uint8_t*)malloc(N);
  if (read_file(argv[6], rgb, 3 * N) || read_file(argv[7], mask, N)) {
    fprintf(stderr, "cannot read the input files\n");
    return 1;
  }
  uint8_t* rgb_d = (uint8_t*)dalloc(3 * N);
  uint8_t* mask_d = (uint8_t*)dalloc(N);
  cudaMemcpy(rgb_d, rgb, 3 * N, cudaMemcpyHostToDevice);
  cudaMemcpy(mask_d, mask, N, cudaMemcpyHostToDevice);

  /* one level (level 1), caller-owned buffers (vinp.h data layout) */
  vinp_level lv;
  memset(&lv, 0, sizeof(lv));
  lv.W = W;
  lv.H = H;
  lv.T = T;
  lv.level = 1;
  lv.vox = (uint64_t*)dalloc(8 * N);
  lv.flags = (uint8_t*)dalloc(N);
  lv.layer = (uint8_t*)dalloc(N);
  lv.slot = (int32_t*)dalloc(4 * N);
  vinp_params prm = {50, -1, 1, 0.5, -1}; /* lambda, tex_half, seed, rho, rmax */

  CK(vinp_build_pyramid(rgb_d, mask_d, &lv, 1, NULL));
  size_t wsb = vinp_texture_ws_bytes(&lv);
  if (vinp_sets_ws_bytes(&lv) > wsb) wsb = vinp_sets_ws_bytes(&lv);
  wsb += 256;
  void* ws = dalloc(wsb);
  CK(vinp_texture_features(&prm, &lv, 1, ws, wsb, NULL));
  int32_t counts[3];
  CK(vinp_build_sets(&lv, 1, counts, ws, wsb, NULL)); /* |H~|, |H|, |D~| (host, synchronises) */
  lv.targets = (int32_t*)dalloc(4 * (size_t)counts[0]);
  lv.holes = (int32_t*)dalloc(4 * (size_t)counts[1]);
  lv.sources = (int32_t*)dalloc(4 * (size_t)counts[2]);
  CK(vinp_build_lists(&lv, 1, ws, wsb, NULL));
  int32_t n_layers = 0;
  CK(vinp_layers(&lv, &n_layers, ws, NULL));

  const int32_t nt = lv.n_targets, nh = lv.n_holes;
  vinp_nnf a, b;
  memset(&a, 0, sizeof(a)); /* mirror = NULL: no peer copies (single process) */
  memset(&b, 0, sizeof(b));
  a.e = (uint64_t*)dalloc(8 * (size_t)nt);
  a.n = (uint8_t*)dalloc((size_t)nt);
  b.e = (uint64_t*)dalloc(8 * (size_t)nt);
  b.n = a.n; /* n is shared by the ping-pong pair */
  a.stamp = (uint8_t*)dalloc((size_t)nt); /* R41 change stamps: one array per buffer */
  b.stamp = (uint8_t*)dalloc((size_t)nt);
  float* cur_rgb = (float*)dalloc(12 * (size_t)nh);
  float* cur_tex = (float*)dalloc(8 * (size_t)nh);
  /* [0] patch-updates (evaluated candidates), [1] stale candidates skipped (R41) */
  unsigned long long* counter = (unsigned long long*)dalloc(16);
  const int32_t steps[4] = {8, 4, 2, 1};

  /* Alg. 4 at the coarsest (= only) level: random phi, onion peel (Alg. 3) */
  CK(vinp_nnf_init_random(&lv, &a, &prm, 0, 0, nt, NULL));
  size_t owsb = vinp_onion_ws_bytes(&lv);
  void* ows = dalloc(owsb);
  CK(vinp_onion_peel(&lv, &a, &b, &prm, K, steps, 4, 0, n_layers, cur_rgb, cur_tex, counter, ows, owsb, NULL));
  for (int k = 0; k < outer; ++k) {
    CK(vinp_ann_search(&lv, &a, &b, &prm, (uint32_t)k, K, steps, 4, 0, -1, -1, counter, NULL));
    CK(vinp_reconstruct(&lv, &a, VINP_WEIGHTED, -1, 0, nh, cur_rgb, cur_tex, 1, NULL));
  }
  CK(vinp_reconstruct(&lv, &a, VINP_BEST_PATCH, -1, 0, nh, cur_rgb, cur_tex, 1, NULL));
  uint8_t* out_d = (uint8_t*)dalloc(3 * N);
  CK(vinp_output_rgb(&lv, out_d, NULL));
  unsigned long long pu[2] = {0, 0};
  cudaMemcpy(pu, counter, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(rgb, out_d, 3 * N, cudaMemcpyDeviceToHost);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  FILE* f = fopen(argv[8], "wb");
  if (!f || fwrite(rgb, 1, 3 * N, f) != 3 * N) {
    fprintf(stderr, "cannot write %s\n", argv[8]);
    return 1;
  }
  fclose(f);
  printf("targets %d holes %d layers %d patch-updates %llu stale-skipped %llu launches %llu\n", nt, nh,
         n_layers, pu[0], pu[1], (unsigned long long)vinp_launch_count());
  return 0;
}
