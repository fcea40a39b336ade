// onion.cu — Alg. 3 onion-peel initialisation at the coarsest level, run natively:
// the layer-j targets and holes are bucketed once into per-layer index lists (stable, ascending),
// then every PatchMatch pass and the Eq. 13 reconstruction of layer j launch over that list only.
// Alg. 3 is strictly sequential over layers, so this turns ~1,700 full-list launches
// into ~1,100 launches over the few thousand indices each layer actually has.
#include <vector>

#include "common.cuh"

namespace vinp {

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }
constexpr int kBT = 256, kBPer = 8, kBChunk = kBT * kBPer, kMaxKeys = 256;

// key(i) = layer[idx[i]]: per-block histogram bc[k * nb + block]
__global__ void k_bucket_count(const int32_t* __restrict__ idx, int32_t n, const uint8_t* __restrict__ layer,
                               int nkeys, int* __restrict__ bc, int nb) {
  __shared__ int h[kMaxKeys];
  for (int k = threadIdx.x; k < nkeys; k += kBT) h[k] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kBChunk;
  for (int r = 0; r < kBPer; ++r) {
    int64_t i = base + r * kBT + threadIdx.x;
    if (i < n) atomicAdd(&h[layer[idx[i]]], 1);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nkeys; k += kBT) bc[k * nb + blockIdx.x] = h[k];
}

// exclusive scan of bc[0..len) (one block)
__global__ void k_bucket_scan(int* __restrict__ a, int len) {
  __shared__ int carry;
  __shared__ int wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < len; base += 1024) {
    int i = base + threadIdx.x;
    int v = i < len ? a[i] : 0;
    int x = v;
    for (int d = 1; d < 32; d <<= 1) {
      int y = __shfl_up_sync(kFull, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = wsum[lane];
      for (int d = 1; d < 32; d <<= 1) {
        int y = __shfl_up_sync(kFull, t, d);
        if (lane >= d) t += y;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    int incl = x + (w ? wsum[w - 1] : 0);
    if (i < len) a[i] = carry + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += incl;
    __syncthreads();
  }
}

// stable scatter: out[offset] = i in ascending i within each key
__global__ void k_bucket_write(const int32_t* __restrict__ idx, int32_t n, const uint8_t* __restrict__ layer,
                               int nkeys, const int* __restrict__ bc, int nb, int32_t* __restrict__ out) {
  __shared__ int run[kMaxKeys];
  __shared__ int wc[kBT / 32][kMaxKeys];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < nkeys; k += kBT) run[k] = bc[k * nb + blockIdx.x];
  for (int k = threadIdx.x; k < (kBT / 32) * kMaxKeys; k += kBT) (&wc[0][0])[k] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kBChunk;
  for (int r = 0; r < kBPer; ++r) {
    int64_t i = base + r * kBT + threadIdx.x;
    int key = i < n ? layer[idx[i]] : -1;
    unsigned peers = __match_any_sync(kFull, key);
    int rank = __popc(peers & ((1u << lane) - 1));
    if (key >= 0 && rank == 0) wc[w][key] = __popc(peers);
    __syncthreads();
    if (key >= 0) {
      int off = run[key];
      for (int w2 = 0; w2 < w; ++w2) off += wc[w2][key];
      out[off + rank] = (int32_t)i;
    }
    __syncthreads();
    if (key >= 0 && rank == 0) {
      // the first lane of each (warp, key) group of the LAST warp holding this key adds the total;
      // simpler: every warp leader adds its own count after everyone has read `run`
      atomicAdd(&run[key], __popc(peers));
    }
    __syncthreads();
    if (key >= 0 && rank == 0) wc[w][key] = 0;
    __syncthreads();
  }
}

// index lists [0, n) of `targets`/`holes` positions bucketed by layer: lists + per-key offsets
static vinp_status bucket(const int32_t* idx, int32_t n, const uint8_t* layer, int nkeys, int32_t* out,
                          int* bc, std::vector<int>& offs, cudaStream_t s) {
  int nb = std::max(1, nblk(n, kBChunk));
  cudaMemsetAsync(bc, 0, sizeof(int) * (size_t)nkeys * nb, s);
  if (n > 0) {
    k_bucket_count<<<nb, kBT, 0, s>>>(idx, n, layer, nkeys, bc, nb);
    k_bucket_scan<<<1, 1024, 0, s>>>(bc, nkeys * nb);
    k_bucket_write<<<nb, kBT, 0, s>>>(idx, n, layer, nkeys, bc, nb, out);
    count_launch(3);
  }
  // per-key start offsets = bc[k * nb + 0] (exclusive scan, key-major)
  offs.assign(nkeys + 1, n);
  std::vector<int> host((size_t)nkeys * nb);
  if (n > 0) {
    if (cudaMemcpyAsync(host.data(), bc, sizeof(int) * host.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return check_launch("vinp_onion_peel(bucket)");
    for (int k = 0; k < nkeys; ++k) offs[k] = host[(size_t)k * nb];
  } else {
    for (int k = 0; k <= nkeys; ++k) offs[k] = 0;
  }
  offs[nkeys] = n;
  return check_launch("vinp_onion_peel(bucket)");
}

__global__ void k_iota(int32_t* a, int32_t n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

// idx indirection for the bucket key: key(i) = layer[targets[i]] / layer[holes[i]]
__global__ void k_gather_layer(const int32_t* __restrict__ pos, int32_t n, const uint8_t* __restrict__ layer,
                               uint8_t* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = layer[pos[i]];
}

}  // namespace vinp

using namespace vinp;

extern "C" {

size_t vinp_onion_ws_bytes(const vinp_level* lv) {
  if (!lv) return 0;
  int64_t nt = lv->n_targets, nh = lv->n_holes;
  int64_t nbt = std::max<int64_t>(1, (nt + kBChunk - 1) / kBChunk), nbh = std::max<int64_t>(1, (nh + kBChunk - 1) / kBChunk);
  return (size_t)(4 * (nt + nh) * 2 + (nt + nh) + 4 * kMaxKeys * (nbt + nbh) + 1024);
}

vinp_status vinp_onion_peel(vinp_level* lv, vinp_nnf* a, vinp_nnf* b, const vinp_params* prm, int K,
                            const int32_t* steps, int n_steps, int sign_policy, int n_layers, float* out_rgb,
                            float* out_tex, unsigned long long* counter, void* ws, size_t ws_bytes,
                            void* stream) {
  VINP_NVTX();
  vinp_status st = check_level(lv, "vinp_onion_peel");
  if (st) return st;
  VINP_REQUIRE(lv->layer && lv->targets && lv->holes && a && b && a->e && b->e && a->e != b->e && prm &&
                   steps && n_steps >= 0 && n_steps <= 16 && K >= 0 && out_rgb && out_tex && ws,
               "vinp_onion_peel: bad arguments");
  VINP_REQUIRE(n_layers >= 0 && n_layers + 1 <= kMaxKeys, "vinp_onion_peel: n_layers out of range");
  VINP_REQUIRE(ws_bytes >= vinp_onion_ws_bytes(lv), "vinp_onion_peel: ws too small");
  cudaStream_t s = S(stream);
  int32_t nt = lv->n_targets, nh = lv->n_holes;
  char* w = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  int32_t* tlist = (int32_t*)w; w += 4 * (size_t)nt;
  int32_t* hlist = (int32_t*)w; w += 4 * (size_t)nh;
  int32_t* iota = (int32_t*)w; w += 4 * (size_t)std::max(nt, nh);
  uint8_t* keys = (uint8_t*)w; w += (size_t)std::max(nt, nh) + 16;
  w = (char*)(((uintptr_t)w + 15) & ~(uintptr_t)15);
  int* bc = (int*)w;
  int nkeys = n_layers + 1;
  int mx = std::max(nt, nh);
  VINP_REQUIRE(!a->stamp == !b->stamp && (!a->stamp || a->stamp != b->stamp),
               "vinp_onion_peel: stamps must be given on both buffers (distinct) or neither");
  vinp_nnf ua = *a, ub = *b;
  const bool use = a->stamp && (int64_t)K * (n_steps + 1) <= 255;
  if (!use) ua.stamp = ub.stamp = nullptr;
  if (mx > 0) {
    k_iota<<<nblk(mx, 256), 256, 0, s>>>(iota, mx);
    count_launch();
  }
  std::vector<int> toff, hoff;
  if (nt > 0) {
    k_gather_layer<<<nblk(nt, 256), 256, 0, s>>>(lv->targets, nt, lv->layer, keys);
    count_launch();
  }
  st = bucket(iota, nt, keys, nkeys, tlist, bc, toff, s);
  if (st) return st;
  if (nh > 0) {
    k_gather_layer<<<nblk(nh, 256), 256, 0, s>>>(lv->holes, nh, lv->layer, keys);
    count_launch();
  }
  st = bucket(iota, nh, keys, nkeys, hlist, bc, hoff, s);
  if (st) return st;

  for (int j = 0; j <= n_layers; ++j) {
    int kb = j < 1 ? 1 : j;
    uint32_t oc = 0x80000000u | (uint32_t)j;
    int tb = toff[j], te = toff[j + 1];
    // both buffers agree outside layer j for the whole layer (Jacobi passes touch layer j only)
    if (nt > 0 && cudaMemcpyAsync(b->e, a->e, 8 * (size_t)nt, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return check_launch("vinp_onion_peel(copy)");
    // R41 stamps: every entry is unchanged since the start of layer j's search (pass 0)
    if (use && nt > 0 && (cudaMemsetAsync(a->stamp, 0, (size_t)nt, s) != cudaSuccess ||
                          cudaMemsetAsync(b->stamp, 0, (size_t)nt, s) != cudaSuccess))
      return check_launch("vinp_onion_peel(stamps)");
    vinp_nnf* cur = &ua;
    vinp_nnf* nxt = &ub;
    if (te > tb) {
      st = launch_evaluate(lv, cur, prm, kb, j, tb, te, tlist, counter, stream);
      if (st) return st;
      PassClock clk;
      for (int k = 1; k <= K; ++k) {
        int sign = sign_policy ? 0 : ((k % 2 == 1) ? 1 : -1);
        for (int i = 0; i < n_steps; ++i) {
          st = launch_propagate(lv, cur, nxt, prm, steps[i], sign, kb, j, tb, te, clk.pass,
                                clk.since(steps[i], sign), tlist, counter, stream);
          if (st) return st;
          clk.tick(steps[i], sign);
          std::swap(cur, nxt);
        }
        st = launch_random_search(lv, cur, nxt, prm, oc, k, kb, j, tb, te, clk.pass, tlist, counter, stream);
        if (st) return st;
        clk.tick(0, 2);
        std::swap(cur, nxt);
      }
      if (cur != &ua && cudaMemcpyAsync(a->e, cur->e, 8 * (size_t)nt, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return check_launch("vinp_onion_peel(copy)");
    }
    if (j >= 1 && hoff[j + 1] > hoff[j]) {
      st = launch_reconstruct(lv, a, VINP_WEIGHTED, j, hoff[j], hoff[j + 1], hlist, out_rgb, out_tex, 1,
                              stream);
      if (st) return st;
    }
  }
  return check_launch("vinp_onion_peel");
}

}  // extern "C"
