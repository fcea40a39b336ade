// alu_bench.cu — SURVEY §8(d): measured issue rate of the patch-distance integer ops on this GPU.
// Each thread runs 8 independent chains of the exact per-voxel sequence of the SSD kernels
// (VABSDIFF4 on the colour word and on the texture word, IDP4A of each with itself accumulated),
// so the loop is throughput-bound, not latency-bound.  Prints G voxel-ops/s (one voxel-op =
// 2 VABSDIFF4 + 2 IDP4A = the work of one patch voxel) and the implied ALU roof in
// patch-updates/s (125 voxel-ops per patch-update).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_bench tools/alu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_alu(const uint32_t* seed, int iters, uint32_t* out) {
  uint32_t t[8], s[8], ac[8], at[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    t[c] = seed[(threadIdx.x + c) & 63] ^ (blockIdx.x * 2654435761u);
    s[c] = seed[(threadIdx.x * 3 + c) & 63];
    ac[c] = 0;
    at[c] = 0;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t dc = __vabsdiffu4(t[c], s[c]);
      uint32_t dt = __vabsdiffu4(t[c] ^ 0x5a5a5a5au, s[c]);
      ac[c] = __dp4a(dc, dc, ac[c]);
      at[c] = __dp4a(dt, dt, at[c]);
      s[c] += ac[c];  // keep the chains live (and data-dependent) without extra loads
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) r += ac[c] * 4u + at[c] * 50u;
  if (r == 0x12345678u) out[0] = r;
}

int main() {
  uint32_t h[64];
  for (int i = 0; i < 64; ++i) h[i] = 0x9e3779b9u * (i + 1);
  uint32_t *d, *o;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 4);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  k_alu<<<blocks, threads>>>(d, 64, o);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_alu<<<blocks, threads>>>(d, iters, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  double vox = (double)blocks * threads * iters * 8;  // voxel-ops
  double rate = vox / (best / 1e3);
  printf("{\"sms\": %d, \"ms\": %.3f, \"G_voxel_ops_per_s\": %.1f, \"G_int_instr_per_s\": %.1f, "
         "\"alu_roof_G_patch_updates_per_s\": %.2f}\n",
         sms, best, rate / 1e9, rate * 5 / 1e9, rate / 125 / 1e9);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
