// encode.cu -- density-aware u8 quantizer on sm_100a (aqr_encode).
//
//   density_kernel      : rho_i = 1/(mean of the k smallest squared L2 distances + eps) over
//                         the density sample, fp64 (Alg1 l.5 at P:114)
//   delta_kernel        : delta = (max rho - min rho)/(max rho + eps) (Alg1 l.6 at P:115),
//                         P_l = delta*P_max, P_h = 100 - delta*P_max (Alg1 l.8 at P:117, R3)
//   transpose_kernel    : X [n x d] -> X^T (column-major) so each column is one contiguous
//                         stream for the selection passes
//   select_kernel       : per dimension, the order statistics at the two percentile ranks by
//                         an 8-bit MSD radix select over order-preserving float keys, then
//                         min_j, max_j, scale_j = 255/(max_j-min_j+eps) (Alg1 l.10-11)
//   encode_kernel       : code = roundf(clamp((x - min_j) * scale_j, 0, 255)) (Alg1 l.9)
//
// Build-time path (once per index, not in the QPS metric).  HBM-bound streaming for the
// transpose/select/encode passes; the density kNN is an fp64 ALU job on an L2-resident sample.
// All floating-point steps use explicitly rounded intrinsics (__dadd_rn, __fmul_rn, ...)
// so no contraction can change a result (compiled with --fmad=false as well).
#include <cfloat>
#include <climits>

#include "aqr_internal.cuh"

namespace aqr {

namespace {

constexpr int kMaxKDensity = 32;

struct DPair {
  double v;
  int32_t id;
};

__device__ __forceinline__ bool dless(double a, int32_t ia, double b, int32_t ib) {
  return a < b || (a == b && ia < ib);
}

// one block per sampled point a; threads stride over the other sample points b
__global__ void __launch_bounds__(256) density_kernel(const float* __restrict__ x, int64_t ld_x, int32_t d,
                                                      const int32_t* __restrict__ sample, int32_t ns,
                                                      int32_t k, double eps, double* __restrict__ rho) {
  extern __shared__ float xi[];
  __shared__ double red_v[8];
  __shared__ int32_t red_i[8];
  __shared__ int32_t red_t[8];
  __shared__ int32_t winner;
  const int a = blockIdx.x;
  const int64_t ia = sample[a];
  for (int t = threadIdx.x; t < d; t += blockDim.x) xi[t] = x[ia * ld_x + t];
  __syncthreads();
  double lv[kMaxKDensity];
  int32_t li[kMaxKDensity];
  int cnt = 0;
  for (int b = threadIdx.x; b < ns; b += blockDim.x) {
    if (b == a) continue;
    const int32_t j = sample[b];
    const float* xj = x + (int64_t)j * ld_x;
    double acc = 0.0;
    for (int t = 0; t < d; ++t) {
      double diff = __dsub_rn((double)xi[t], (double)__ldg(xj + t));
      acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    // keep this thread's k smallest (value, id), ascending
    if (cnt < k || dless(acc, j, lv[cnt - 1], li[cnt - 1])) {
      int p = cnt < k ? cnt : k - 1;
      while (p > 0 && dless(acc, j, lv[p - 1], li[p - 1])) {
        lv[p] = lv[p - 1];
        li[p] = li[p - 1];
        --p;
      }
      lv[p] = acc;
      li[p] = j;
      if (cnt < k) ++cnt;
    }
  }
  // k rounds of block-wide argmin over the per-thread heads; thread 0 sums ascending
  int head = 0;
  double s = 0.0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = 0; r < k; ++r) {
    double v = head < cnt ? lv[head] : DBL_MAX;
    int32_t id = head < cnt ? li[head] : INT_MAX;
    int32_t tid = threadIdx.x;
    for (int off = 16; off; off >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, v, off);
      int32_t oi = __shfl_xor_sync(0xffffffffu, id, off);
      int32_t ot = __shfl_xor_sync(0xffffffffu, tid, off);
      if (dless(ov, oi, v, id)) { v = ov; id = oi; tid = ot; }
    }
    if (lane == 0) { red_v[w] = v; red_i[w] = id; red_t[w] = tid; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bv = red_v[0];
      int32_t bi = red_i[0], bt = red_t[0];
      for (int q = 1; q < nw; ++q)
        if (dless(red_v[q], red_i[q], bv, bi)) { bv = red_v[q]; bi = red_i[q]; bt = red_t[q]; }
      s = __dadd_rn(s, bv);
      winner = bt;
    }
    __syncthreads();
    if (threadIdx.x == winner) ++head;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double mean = __ddiv_rn(s, (double)k);
    rho[a] = __ddiv_rn(1.0, __dadd_rn(mean, eps));
  }
}

__global__ void delta_kernel(const double* __restrict__ rho, int32_t ns, double eps, double delta_override,
                             double p_max, double* __restrict__ meta) {
  __shared__ double smx[32], smn[32];
  double mx = -DBL_MAX, mn = DBL_MAX;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    mx = fmax(mx, rho[i]);
    mn = fmin(mn, rho[i]);
  }
  for (int off = 16; off; off >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
  }
  if ((threadIdx.x & 31) == 0) { smx[threadIdx.x >> 5] = mx; smn[threadIdx.x >> 5] = mn; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { mx = fmax(mx, smx[w]); mn = fmin(mn, smn[w]); }
    mx = fmax(mx, smx[0]);
    mn = fmin(mn, smn[0]);
    double delta = isnan(delta_override) ? __ddiv_rn(__dsub_rn(mx, mn), __dadd_rn(mx, eps)) : delta_override;
    double dp = __dmul_rn(delta, p_max);
    meta[0] = delta;
    meta[1] = dp;
    meta[2] = __dsub_rn(100.0, dp);
  }
}

__global__ void delta_only_kernel(double delta, double p_max, double* meta) {
  double dp = __dmul_rn(delta, p_max);
  meta[0] = delta;
  meta[1] = dp;
  meta[2] = __dsub_rn(100.0, dp);
}

__global__ void transpose_kernel(const float* __restrict__ x, int64_t n, int32_t d, int64_t ld_x,
                                 float* __restrict__ xt) {
  __shared__ float tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int j0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t i = i0 + r;
    int j = j0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < n && j < d) ? x[i * ld_x + j] : 0.0f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int j = j0 + r;
    int64_t i = i0 + threadIdx.x;
    if (j < d && i < n) xt[(int64_t)j * n + i] = tile[threadIdx.x][r];
  }
}

__device__ __forceinline__ uint32_t fkey(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k ^ 0x80000000u) : ~k;
  return __uint_as_float(u);
}

// rank of percentile P (percent scale) in a sorted array of n: r = (P/100)(n-1), lo, hi, f
__device__ __forceinline__ void pct_rank(double P, int64_t n, int64_t& lo, int64_t& hi, double& f) {
  double r = __dmul_rn(__ddiv_rn(P, 100.0), (double)(n - 1));
  lo = (int64_t)floor(r);
  if (lo < 0) lo = 0;
  if (lo > n - 1) lo = n - 1;
  hi = (lo + 1 < n - 1) ? lo + 1 : n - 1;
  f = __dsub_rn(r, (double)lo);
}

// one block per dimension: 4 radix-select targets (lo/hi rank of P_l and of P_h)
__global__ void __launch_bounds__(1024) select_kernel(const float* __restrict__ xt, int64_t n,
                                                     const double* __restrict__ meta, double eps,
                                                     float* __restrict__ min_j, float* __restrict__ max_j,
                                                     float* __restrict__ scale_j) {
  __shared__ uint32_t hist[4][256];
  __shared__ uint32_t prefix[4];
  __shared__ int64_t want[4];
  __shared__ double fr[2];
  const int j = blockIdx.x;
  const float* col = xt + (int64_t)j * n;
  if (threadIdx.x == 0) {
    int64_t lo, hi;
    double f;
    pct_rank(meta[1], n, lo, hi, f);
    want[0] = lo; want[1] = hi; fr[0] = f;
    pct_rank(meta[2], n, lo, hi, f);
    want[2] = lo; want[3] = hi; fr[1] = f;
    for (int t = 0; t < 4; ++t) prefix[t] = 0;
  }
  __syncthreads();
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    const uint32_t mask = pass == 0 ? 0u : (0xFFFFFFFFu << (32 - 8 * pass));
    for (int t = threadIdx.x; t < 4 * 256; t += blockDim.x) (&hist[0][0])[t] = 0;
    __syncthreads();
    uint32_t p0 = prefix[0], p1 = prefix[1], p2 = prefix[2], p3 = prefix[3];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      uint32_t key = fkey(col[i]);
      uint32_t km = key & mask;
      uint32_t b = (key >> shift) & 255u;
      if (km == p0) atomicAdd(&hist[0][b], 1u);
      if (km == p1) atomicAdd(&hist[1][b], 1u);
      if (km == p2) atomicAdd(&hist[2][b], 1u);
      if (km == p3) atomicAdd(&hist[3][b], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 4) {
      const int t = threadIdx.x;
      int64_t r = want[t];
      uint32_t b = 0;
      for (; b < 256; ++b) {
        if (r < (int64_t)hist[t][b]) break;
        r -= hist[t][b];
      }
      want[t] = r;
      prefix[t] |= (b << shift);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double s0 = (double)fkey_inv(prefix[0]), s1 = (double)fkey_inv(prefix[1]);
    double s2 = (double)fkey_inv(prefix[2]), s3 = (double)fkey_inv(prefix[3]);
    double mn = __dadd_rn(s0, __dmul_rn(fr[0], __dsub_rn(s1, s0)));
    double mx = __dadd_rn(s2, __dmul_rn(fr[1], __dsub_rn(s3, s2)));
    double range = __dsub_rn(mx, mn);
    min_j[j] = __double2float_rn(mn);
    max_j[j] = __double2float_rn(mx);
    scale_j[j] = range < 1e-9 ? 1.0f : __double2float_rn(__ddiv_rn(255.0, __dadd_rn(range, eps)));
  }
}

__device__ __forceinline__ uint32_t quant1(float xv, float mn, float sc) {
  float t = __fsub_rn(xv, mn);
  float u = __fmul_rn(t, sc);
  float v = fminf(fmaxf(u, 0.0f), 255.0f);
  return (uint32_t)roundf(v);
}

// one thread per 16-byte output chunk of a code row
__global__ void encode_kernel(const float* __restrict__ x, int64_t n, int32_t d, int64_t ld_x,
                              const float* __restrict__ mn, const float* __restrict__ sc,
                              uint8_t* __restrict__ codes, int32_t d_pad) {
  const int nch = d_pad >> 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = tid / nch;
  const int c = (int)(tid - i * nch);
  if (i >= n) return;
  const float* row = x + i * ld_x;
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int j = c * 16 + q * 4 + b;
      uint32_t code = 0;
      if (j < d) code = quant1(__ldg(row + j), __ldg(mn + j), __ldg(sc + j));
      v |= code << (8 * b);
    }
    w[q] = v;
  }
  reinterpret_cast<uint4*>(codes + i * d_pad)[c] = make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace

cudaError_t launch_density(const float* x, int64_t ld_x, int32_t d, const int32_t* sample, int32_t ns,
                           int32_t k, double eps, double* rho, cudaStream_t s) {
  if (k > kMaxKDensity) return cudaErrorInvalidValue;
  size_t smem = sizeof(float) * (size_t)d;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(density_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  density_kernel<<<ns, 256, smem, s>>>(x, ld_x, d, sample, ns, k, eps, rho);
  return cudaGetLastError();
}

cudaError_t launch_delta(const double* rho, int32_t ns, double eps, double delta_override, double p_max,
                         double* meta, cudaStream_t s) {
  if (rho == nullptr) {
    delta_only_kernel<<<1, 1, 0, s>>>(delta_override, p_max, meta);
  } else {
    delta_kernel<<<1, 1024, 0, s>>>(rho, ns, eps, delta_override, p_max, meta);
  }
  return cudaGetLastError();
}

cudaError_t launch_train_columns(const float* x, int64_t n, int32_t d, int64_t ld_x, const double* meta,
                                 double eps, float* min_j, float* max_j, float* scale_j, void* tmp,
                                 cudaStream_t s) {
  float* xt = static_cast<float*>(tmp);
  dim3 tb(32, 8);
  dim3 tg((unsigned)((n + 31) / 32), (unsigned)((d + 31) / 32));
  transpose_kernel<<<tg, tb, 0, s>>>(x, n, d, ld_x, xt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  select_kernel<<<d, 1024, 0, s>>>(xt, n, meta, eps, min_j, max_j, scale_j);
  return cudaGetLastError();
}

cudaError_t launch_encode(const float* x, int64_t n, int32_t d, int64_t ld_x, const float* min_j,
                          const float* scale_j, uint8_t* codes, int32_t d_pad, cudaStream_t s) {
  const int64_t total = n * (int64_t)(d_pad >> 4);
  const int bs = 256;
  const int64_t grid = (total + bs - 1) / bs;
  encode_kernel<<<(unsigned)grid, bs, 0, s>>>(x, n, d, ld_x, min_j, scale_j, codes, d_pad);
  return cudaGetLastError();
}

}  // namespace aqr
