// merge.cu -- cross-shard top-k merge (aqr_merge_topk), BASELINE.json configs[4]:
// "per-shard top-k gathered over NVLink and merged".  One warp per query; lane s holds the
// head of list s (n_lists <= 32); k rounds of a warp-wide (dist, id) argmin.
#include "aqr_internal.cuh"

namespace aqr {

namespace {

__device__ __forceinline__ uint64_t mkey(float d, int32_t id) {
  uint32_t u = __float_as_uint(d);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((uint64_t)u << 32) | (uint32_t)id;
}

__global__ void __launch_bounds__(256) merge_kernel(const float* __restrict__ dist, const int32_t* __restrict__ ids,
                                                    int32_t n_lists, int64_t nq, int32_t k,
                                                    float* __restrict__ out_dist, int32_t* __restrict__ out_ids) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (qi >= nq) return;
  int head = 0;
  const int64_t base = ((int64_t)lane * nq + qi) * k;
  for (int t = 0; t < k; ++t) {
    uint64_t key = ~0ull;
    if (lane < n_lists && head < k) {
      const int32_t id = __ldg(ids + base + head);
      if (id >= 0) key = mkey(__ldg(dist + base + head), id);
    }
    uint64_t best = key;
#pragma unroll
    for (int m = 16; m; m >>= 1) {
      uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)best, m);
      uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(best >> 32), m);
      uint64_t o = ((uint64_t)hi << 32) | lo;
      best = o < best ? o : best;
    }
    if (best == ~0ull) {
      for (int r = t + lane; r < k; r += 32) {
        out_ids[qi * k + r] = -1;
        out_dist[qi * k + r] = INFINITY;
      }
      break;
    }
    if (key == best) ++head;  // (dist, id) keys are distinct across lists
    if (lane == 0) {
      const uint32_t u = (uint32_t)(best >> 32);
      out_dist[qi * k + t] = __uint_as_float((u & 0x80000000u) ? (u ^ 0x80000000u) : ~u);
      out_ids[qi * k + t] = (int32_t)(uint32_t)best;
    }
  }
}

}  // namespace

cudaError_t launch_merge(const float* dist, const int32_t* ids, int32_t n_lists, int64_t nq, int32_t k,
                         float* out_dist, int32_t* out_ids, cudaStream_t s) {
  const int wpb = 8;
  const int64_t grid = (nq + wpb - 1) / wpb;
  merge_kernel<<<(unsigned)grid, wpb * 32, 0, s>>>(dist, ids, n_lists, nq, k, out_dist, out_ids);
  return cudaGetLastError();
}

}  // namespace aqr
