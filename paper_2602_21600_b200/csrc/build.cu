// build.cu -- GPU index build: HNSW insertion over the quantized codes (Alg1 l.16-22, P:125-131;
// SURVEY 8(f) NEXT-1), behind aqr_build_graph (include/aqr.h).
//
// The graph is byte-identical to the oracle's or_build_graph and to the host builder
// (csrc/hnsw_build.cpp): same insertion order (R28 "waves"), same integer distances
// d^q with (d, id) ties, same SEARCH-LAYER result (flag form), same neighbour
// selection (Malkov's heuristic, R14).  Per wave (batch of B new nodes, in id order):
//   1. insert_kernel -- one warp per new node, on the graph as it stood when the wave began
//      (no node of the wave is linked yet): greedy descent above the node's level, then at each
//      layer <= level an ef_c beam started from the previous layer's W, the heuristic selection,
//      the node's own row, and one 48-bit key (layer, target, node) per reverse link into its
//      fixed slot range (unused slots = ~0);
//   2. cub radix sort of the wave's keys -> (layer, target) groups, sources in id order;
//   3. group_kernel -- one warp per group: append the sources to the target row, or, when the
//      row overflows, re-select it by the heuristic over (row + sources) sorted by (d^q, id).
// The wave sizes and the entry point / top level follow from the levels alone, so the host
// drives the waves without reading anything back.
//
// d^q of a code row against a list of rows: LPR lanes per row, one 256-bit load per lane and
// 32-byte chunk, dp4a, |x^|^2 precomputed per node (exact int32), as in the search kernel.
#include <cub/cub.cuh>

#include <climits>
#include <vector>

#include "aqr_internal.cuh"

namespace aqr {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kCapMax = 160;   // layer-0 rows (2M, M <= 80)
constexpr int kWaveMax = 4096;  // nodes per wave (R28)
constexpr uint64_t kNoKey = ~0ull;

struct BView {
  const uint8_t* codes;   // [n x d_pad], d_pad a multiple of 32, zero padded
  const int32_t* xnorm;   // [n] |x^|^2
  int32_t d_pad, M, cap0;
  int32_t* adj0;          // [n x cap0]
  int32_t* adj_up;        // [upper rows x M]
  const int32_t* up_off;  // [n] row of (v, layer 1), -1 for level-0 nodes
  const int32_t* levels;  // [n]
};

__device__ __forceinline__ int32_t* brow(const BView& g, int64_t v, int L) {
  return L == 0 ? g.adj0 + v * g.cap0 : g.adj_up + ((int64_t)g.up_off[v] + L - 1) * g.M;
}

struct C32 {
  uint4 a, b;
};

__device__ __forceinline__ void ldg256(const void* p, C32& v) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.a.x), "=r"(v.a.y), "=r"(v.a.z), "=r"(v.a.w), "=r"(v.b.x), "=r"(v.b.y), "=r"(v.b.z),
                 "=r"(v.b.w)
               : "l"(p));
}

__device__ __forceinline__ uint32_t dot8(const C32& w, const C32& q, uint32_t acc) {
  acc = __dp4a(q.a.x, w.a.x, acc);
  acc = __dp4a(q.a.y, w.a.y, acc);
  acc = __dp4a(q.a.z, w.a.z, acc);
  acc = __dp4a(q.a.w, w.a.w, acc);
  acc = __dp4a(q.b.x, w.b.x, acc);
  acc = __dp4a(q.b.y, w.b.y, acc);
  acc = __dp4a(q.b.z, w.b.z, acc);
  return __dp4a(q.b.w, w.b.w, acc);
}

__device__ __forceinline__ uint64_t key_of(uint32_t d, int32_t id) { return ((uint64_t)d << 32) | (uint32_t)id; }
__device__ __forceinline__ int32_t key_id(uint64_t k) { return (int32_t)(uint32_t)k; }
__device__ __forceinline__ uint32_t key_d(uint64_t k) { return (uint32_t)(k >> 32); }

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  const uint32_t hi = (uint32_t)(v >> 32);
  const uint32_t mh = __reduce_min_sync(kFull, hi);
  const uint32_t ml = __reduce_min_sync(kFull, hi == mh ? (uint32_t)v : 0xffffffffu);
  return ((uint64_t)mh << 32) | ml;
}

// the "query" of a distance list: one node's code row spread over the lanes (lane sub of a row
// group owns chunks sub + LPR t), and |q^|^2
template <int LPR, int CPL>
struct QRow {
  C32 r[CPL];
  int32_t qq;
  __device__ void load(const BView& g, int64_t v, int lane) {
    const int sub = lane % LPR, nch = g.d_pad >> 5;
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int c = sub + LPR * t;
      if (c < nch) {
        ldg256(g.codes + v * g.d_pad + 32 * c, r[t]);
      } else {
        r[t].a = make_uint4(0, 0, 0, 0);
        r[t].b = make_uint4(0, 0, 0, 0);
      }
    }
    qq = __ldg(g.xnorm + v);
  }
};

// d^q from q to ids[0 .. m) (entries < 0 give INT_MAX) into out[0 .. m); rows of U per lane group
template <int LPR, int CPL>
__device__ void dist_list(const BView& g, const QRow<LPR, CPL>& q, const int32_t* ids, int m, int32_t* out, int lane) {
  constexpr int G = 32 / LPR;
  constexpr int U = 8;
  const int grp = lane / LPR, sub = lane % LPR;
  const int nch = g.d_pad >> 5;
  for (int r0 = 0; r0 < m; r0 += G * U) {
    C32 buf[U][CPL];
    int idv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + grp * U + u;
      idv[u] = r < m ? ids[r] : -1;
      const uint8_t* row = g.codes + (int64_t)(idv[u] < 0 ? 0 : idv[u]) * g.d_pad;
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = sub + LPR * t;
        if (idv[u] >= 0 && c < nch) {
          ldg256(row + 32 * c, buf[u][t]);
        } else {
          buf[u][t].a = make_uint4(0, 0, 0, 0);
          buf[u][t].b = make_uint4(0, 0, 0, 0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t dot = 0;
#pragma unroll
      for (int t = 0; t < CPL; ++t) dot = dot8(buf[u][t], q.r[t], dot);
      // reduce over the LPR lanes of the row group
#pragma unroll
      for (int o = LPR / 2; o >= 1; o >>= 1) dot += __shfl_xor_sync(kFull, dot, o);
      const int r = r0 + grp * U + u;
      if (sub == 0 && r < m)
        out[r] = idv[u] >= 0 ? q.qq + __ldg(g.xnorm + idv[u]) - 2 * (int32_t)dot : INT_MAX;
    }
  }
  __syncwarp();
}

// rank sort of n distinct 64-bit keys from src into dst (ascending)
__device__ void rank_sort(const uint64_t* src, uint64_t* dst, int n, int lane) {
  for (int i = lane; i < n; i += 32) {
    const uint64_t k = src[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += src[j] < k;
    dst[r] = k;
  }
  __syncwarp();
}

// Malkov's heuristic (R14) over cand[0 .. nc) sorted by (d, id) (d = d^q to the base node): keep e
// unless a kept r has d^q(e, r) < d(e); stop at m kept; keep_pruned fills the free slots with the
// rejected ones in scan order.  sel / pruned / dtmp: shared scratch.  Returns the count kept.
template <int LPR, int CPL>
__device__ int select_heuristic(const BView& g, const uint64_t* cand, int nc, int m, bool keep_pruned, int32_t* sel,
                                int32_t* pruned, int32_t* dtmp, int lane) {
  int ns = 0, np = 0;
  for (int i = 0; i < nc && ns < m; ++i) {
    const int32_t e = key_id(cand[i]);
    const int32_t de = (int32_t)key_d(cand[i]);
    bool good = true;
    if (ns > 0) {
      QRow<LPR, CPL> qe;
      qe.load(g, e, lane);
      dist_list<LPR, CPL>(g, qe, sel, ns, dtmp, lane);
      bool closer = false;
      for (int j = lane; j < ns; j += 32) closer |= dtmp[j] < de;
      good = __ballot_sync(kFull, closer) == 0;
    }
    if (lane == 0) {
      if (good) sel[ns] = e;
      else if (keep_pruned) pruned[np] = e;
    }
    if (good) ++ns;
    else if (keep_pruned) ++np;
    __syncwarp();
  }
  for (int i = 0; i < np && ns < m; ++i) {
    if (lane == 0) sel[ns] = pruned[i];
    ++ns;
  }
  __syncwarp();
  return ns;
}

// per-warp shared memory of insert_kernel
struct ILayout {
  int o_w, o_w2, o_nb, o_nd, o_cand, o_cs, o_sel, o_pr, bytes;
};
__host__ __device__ inline ILayout ilayout(int efc) {
  ILayout L;
  int o = 0;
  auto al = [](int x) { return (x + 15) & ~15; };
  L.o_w = o; o += al(8 * (efc + 1));
  L.o_w2 = o; o += al(8 * (efc + 1));
  L.o_nb = o; o += al(4 * (kCapMax + 32));
  L.o_nd = o; o += al(4 * (kCapMax + 32));
  L.o_cand = o; o += al(8 * kCapMax);
  L.o_cs = o; o += al(8 * kCapMax);
  L.o_sel = o; o += al(4 * kCapMax);
  L.o_pr = o; o += al(4 * (efc + kCapMax));
  L.bytes = (o + 127) & ~127;
  return L;
}

// The flag-form beam (R8) at layer L from W[0 .. size) (all unexpanded): W holds
// keys (d^q << 32 | id) in ascending order, the expanded flag in bit 31 of the id word (ids <
// 2^31).  Re-encountered nodes are re-scored and dropped against W (A.3).  Returns the size.
__device__ __forceinline__ bool expanded(uint64_t k) { return (k & 0x80000000ull) != 0; }
__device__ __forceinline__ uint64_t strip(uint64_t k) { return k & ~0x80000000ull; }

template <int LPR, int CPL>
__device__ int beam(const BView& g, const QRow<LPR, CPL>& q, int L, int ef, uint64_t* W, int size, uint64_t* W2,
                    int32_t* nb, int32_t* nd, uint64_t* cand, uint64_t* cs, int lane) {
  const int cap = L == 0 ? g.cap0 : g.M;
  int cursor = 0;
  for (;;) {
    int pos = -1;
    for (int b = cursor; b < size; b += 32) {
      const int i = b + lane;
      const uint32_t mk = __ballot_sync(kFull, i < size && !expanded(W[i]));
      if (mk) { pos = b + __ffs(mk) - 1; break; }
    }
    if (pos < 0) break;
    const int32_t c = key_id(strip(W[pos]));
    __syncwarp();
    if (lane == 0) W[pos] |= 0x80000000ull;
    cursor = pos + 1;
    // the row (packed; it ends at its first -1)
    const int32_t* row = brow(g, c, L);
    int m = 0;
    for (int t0 = 0; t0 < cap; t0 += 32) {
      const int32_t u = t0 + lane < cap ? row[t0 + lane] : -1;
      const uint32_t mk = __ballot_sync(kFull, u >= 0);
      if (u >= 0) nb[m + __popc(mk & ((1u << lane) - 1u))] = u;
      m += __popc(mk);
    }
    __syncwarp();
    dist_list<LPR, CPL>(g, q, nb, m, nd, lane);
    // filter against max W, drop nodes already in W (re-evaluations)
    const uint64_t maxk = size >= ef ? strip(W[size - 1]) : kNoKey;
    int np = 0;
    for (int r0 = 0; r0 < m; r0 += 32) {
      const int r = r0 + lane;
      bool ok = false;
      uint64_t kk = 0;
      if (r < m) {
        kk = key_of((uint32_t)nd[r], nb[r]);
        ok = kk < maxk;
        if (ok) {
          int lo = 0, hi = size;  // lower bound of kk in W (flag bit ignored)
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (strip(W[mid]) < kk) lo = mid + 1;
            else hi = mid;
          }
          ok = !(lo < size && strip(W[lo]) == kk);
        }
      }
      const uint32_t mk = __ballot_sync(kFull, ok);
      if (ok) cand[np + __popc(mk & ((1u << lane) - 1u))] = kk;
      np += __popc(mk);
    }
    __syncwarp();
    if (np == 0) continue;
    rank_sort(cand, cs, np, lane);
    // merge W and cs (both ascending) into W2, keep the first ef, swap back
    const int total = size + np < ef ? size + np : ef;
    for (int i = lane; i < size; i += 32) {
      const uint64_t k = W[i], ks = strip(k);
      int r = 0;
      while (r < np && cs[r] < ks) ++r;
      if (i + r < ef) W2[i + r] = k;
    }
    for (int j = lane; j < np; j += 32) {
      const uint64_t k = cs[j];
      int lo = 0, hi = size;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (strip(W[mid]) < k) lo = mid + 1;
        else hi = mid;
      }
      if (lo + j < ef) W2[lo + j] = k;
    }
    __syncwarp();
    for (int i = lane; i < total; i += 32) W[i] = W2[i];
    __syncwarp();
    // the smallest unexpanded entry can now sit before the cursor (a new key)
    const uint64_t c0 = cs[0];
    int lb = 0, hi = total;
    while (lb < hi) {
      const int mid = (lb + hi) >> 1;
      if (strip(W[mid]) < c0) lb = mid + 1;
      else hi = mid;
    }
    if (lb < cursor) cursor = lb;
    size = total;
  }
  return size;
}

template <int LPR, int CPL>
__global__ void __launch_bounds__(128) insert_kernel(BView g, int64_t pos, int32_t B, int32_t entry, int32_t max_level,
                                                     int32_t efc, int32_t sel0, int32_t keep_pruned,
                                                     const int64_t* __restrict__ slot_off, uint64_t* __restrict__ keys) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int bi = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (bi >= B) return;
  const ILayout Ly = ilayout(efc);
  uint8_t* wb = smem + (threadIdx.x >> 5) * Ly.bytes;
  uint64_t* W = reinterpret_cast<uint64_t*>(wb + Ly.o_w);
  uint64_t* W2 = reinterpret_cast<uint64_t*>(wb + Ly.o_w2);
  int32_t* nb = reinterpret_cast<int32_t*>(wb + Ly.o_nb);
  int32_t* nd = reinterpret_cast<int32_t*>(wb + Ly.o_nd);
  uint64_t* cand = reinterpret_cast<uint64_t*>(wb + Ly.o_cand);
  uint64_t* cs = reinterpret_cast<uint64_t*>(wb + Ly.o_cs);
  int32_t* sel = reinterpret_cast<int32_t*>(wb + Ly.o_sel);
  int32_t* pr = reinterpret_cast<int32_t*>(wb + Ly.o_pr);
  const int64_t qn = pos + bi;
  const int lq = g.levels[qn];
  QRow<LPR, CPL> q;
  q.load(g, qn, lane);
  // greedy descent through the layers above the node's level (O9)
  int32_t cur = entry;
  if (lane == 0) nb[0] = cur;
  __syncwarp();
  dist_list<LPR, CPL>(g, q, nb, 1, nd, lane);
  uint32_t dcur = (uint32_t)nd[0];
  __syncwarp();
  for (int L = max_level; L > lq; --L) {
    for (;;) {
      const int32_t* row = brow(g, cur, L);
      int m = 0;
      for (int t0 = 0; t0 < g.M; t0 += 32) {
        const int32_t u = t0 + lane < g.M ? row[t0 + lane] : -1;
        const uint32_t mk = __ballot_sync(kFull, u >= 0);
        if (u >= 0) nb[m + __popc(mk & ((1u << lane) - 1u))] = u;
        m += __popc(mk);
      }
      __syncwarp();
      dist_list<LPR, CPL>(g, q, nb, m, nd, lane);
      uint64_t best = key_of(dcur, cur);
      for (int r = lane; r < m; r += 32) {
        const uint64_t kk = key_of((uint32_t)nd[r], nb[r]);
        best = kk < best ? kk : best;
      }
      best = warp_min_u64(best);
      __syncwarp();
      if (key_id(best) == cur) break;
      cur = key_id(best);
      dcur = key_d(best);
    }
  }
  // layers min(lq, max_level) .. 0: beam from the previous layer's W (all unexpanded), select,
  // write the node's own row, emit the reverse-link keys
  int size = 1;
  if (lane == 0) W[0] = key_of(dcur, cur);
  __syncwarp();
  uint64_t* out = keys + slot_off[bi];
  int nout = 0;
  const int top = lq < max_level ? lq : max_level;
  for (int L = top; L >= 0; --L) {
    for (int i = lane; i < size; i += 32) W[i] = strip(W[i]);
    __syncwarp();
    size = beam<LPR, CPL>(g, q, L, efc, W, size, W2, nb, nd, cand, cs, lane);
    for (int i = lane; i < size; i += 32) W2[i] = strip(W[i]);  // sorted candidates for the selection
    __syncwarp();
    const int m = select_heuristic<LPR, CPL>(g, W2, size, L == 0 ? sel0 : g.M, keep_pruned != 0, sel, pr, nd, lane);
    int32_t* row = brow(g, qn, L);
    for (int t = lane; t < m; t += 32) {
      row[t] = sel[t];
      // (layer, target, position in the wave): 5 + 31 + 12 bits, sorted by layer, target, source
      out[nout + t] = ((uint64_t)L << 43) | ((uint64_t)(uint32_t)sel[t] << 12) | (uint64_t)bi;
    }
    nout += m;
    __syncwarp();
  }
  const int nslots = (int)(slot_off[bi + 1] - slot_off[bi]);
  for (int t = nout + lane; t < nslots; t += 32) out[t] = kNoKey;
}

// group heads of the sorted keys: one entry per (layer, target)
__global__ void heads_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ heads,
                             int32_t* __restrict__ nheads) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  if (k == kNoKey) return;
  if (i == 0 || (keys[i - 1] >> 12) != (k >> 12)) heads[atomicAdd(nheads, 1)] = i;
}

template <int LPR, int CPL>
__global__ void __launch_bounds__(128) group_kernel(BView g, int64_t pos, const uint64_t* __restrict__ keys,
                                                    int64_t nkeys, const int64_t* __restrict__ heads,
                                                    const int32_t* __restrict__ nheads, int32_t keep_pruned,
                                                    uint64_t* __restrict__ scratch, int64_t scratch_per_warp) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  uint8_t* wb = smem + (threadIdx.x >> 5) * (4 * kCapMax * 2 + 64);
  int32_t* sel = reinterpret_cast<int32_t*>(wb);
  int32_t* dtmp = sel + kCapMax;
  // per-warp global scratch for a group of up to NC = cap0 + wave + 64 candidates
  const int64_t NC = scratch_per_warp / 4;
  uint64_t* cbuf = scratch + wid * scratch_per_warp;  // [NC] candidates, unsorted
  uint64_t* sbuf = cbuf + NC;                          // [NC] sorted
  int32_t* ibuf = reinterpret_cast<int32_t*>(sbuf + NC);  // [NC] ids for dist_list
  int32_t* dbuf = ibuf + NC;                              // [NC] their d^q
  int32_t* pr = dbuf + NC;                                // [NC] rejected ids (keep_pruned)
  const int ng = *nheads;
  for (int64_t gi = wid; gi < ng; gi += nw) {
    const int64_t a = heads[gi];
    const uint64_t head = keys[a] >> 12;
    int64_t b = a + 1;
    while (b < nkeys && (keys[b] >> 12) == head) ++b;
    const int L = (int)(keys[a] >> 43);
    const int32_t e = (int32_t)((keys[a] >> 12) & 0x7fffffffull);
    const int cap = L == 0 ? g.cap0 : g.M;
    int32_t* row = brow(g, e, L);
    int deg = 0;
    for (int t0 = 0; t0 < cap; t0 += 32) deg += __popc(__ballot_sync(kFull, t0 + lane < cap && row[t0 + lane] >= 0));
    const int cnt = (int)(b - a);
    if (deg + cnt <= cap) {
      for (int i = lane; i < cnt; i += 32) row[deg + i] = (int32_t)(pos + (int64_t)(keys[a + i] & 0xfffull));
      __syncwarp();
      continue;
    }
    // overflow: re-select the row from (old row + new sources) by (d^q to e, id)
    const int nc = deg + cnt;
    for (int i = lane; i < nc; i += 32)
      ibuf[i] = i < deg ? row[i] : (int32_t)(pos + (int64_t)(keys[a + i - deg] & 0xfffull));
    __syncwarp();
    QRow<LPR, CPL> qe;
    qe.load(g, e, lane);
    dist_list<LPR, CPL>(g, qe, ibuf, nc, dbuf, lane);
    for (int i = lane; i < nc; i += 32) cbuf[i] = key_of((uint32_t)dbuf[i], ibuf[i]);
    __syncwarp();
    rank_sort(cbuf, sbuf, nc, lane);
    const int m = select_heuristic<LPR, CPL>(g, sbuf, nc, cap, keep_pruned != 0, sel, pr, dtmp, lane);
    for (int t = lane; t < cap; t += 32) row[t] = t < m ? sel[t] : -1;
    __syncwarp();
  }
}

struct Shape {
  int lpr, cpl;
};
Shape shape_of(int d_pad) {
  const int nch = d_pad >> 5;
  int lpr = 1;
  while (lpr < nch) lpr <<= 1;
  if (lpr > 32) lpr = 32;
  return Shape{lpr, (nch + lpr - 1) / lpr};
}

template <int LPR, int CPL>
cudaError_t run_waves(const BView& g, int64_t n, const int32_t* levels_h, int32_t efc, int32_t sel0,
                      int32_t keep_pruned, int32_t batch_div, int32_t* entry_max, cudaStream_t s) {
  // slot ranges per node (max reverse links it can emit: sel0 at layer 0, M per layer above, up
  // to the top level when its wave begins), and the waves themselves, from the levels alone
  std::vector<int64_t> wave_lo;
  std::vector<int32_t> wave_entry, wave_top;
  int32_t entry = 0, top = levels_h[0];
  int64_t max_slots = 0;
  for (int64_t p = 1; p < n;) {
    int64_t B = p / batch_div;
    B = B < 1 ? 1 : (B > kWaveMax ? kWaveMax : B);
    if (B > n - p) B = n - p;
    for (int64_t i = 0; i < B; ++i)
      if (levels_h[p + i] > top) { B = i == 0 ? 1 : i; break; }
    wave_lo.push_back(p);
    wave_entry.push_back(entry);
    wave_top.push_back(top);
    int64_t acc = 0;
    for (int64_t i = 0; i < B; ++i) {
      const int lq = levels_h[p + i] < top ? levels_h[p + i] : top;
      acc += sel0 + (int64_t)g.M * lq;
    }
    max_slots = acc > max_slots ? acc : max_slots;
    for (int64_t i = 0; i < B; ++i)
      if (levels_h[p + i] > top) { top = levels_h[p + i]; entry = (int32_t)(p + i); }
    p += B;
  }
  wave_lo.push_back(n);
  // per-wave relative slot offsets [B + 1] each, packed back to back
  std::vector<int64_t> off_h;
  std::vector<int64_t> off_at;
  for (size_t w = 0; w + 1 < wave_lo.size(); ++w) {
    const int64_t p = wave_lo[w], B = wave_lo[w + 1] - p;
    off_at.push_back((int64_t)off_h.size());
    int64_t acc = 0;
    for (int64_t i = 0; i < B; ++i) {
      off_h.push_back(acc);
      const int lq = levels_h[p + i] < wave_top[w] ? levels_h[p + i] : wave_top[w];
      acc += sel0 + (int64_t)g.M * lq;
    }
    off_h.push_back(acc);
  }
  int64_t* off_d = nullptr;
  uint64_t *keys = nullptr, *keys2 = nullptr, *scratch = nullptr;
  int64_t* heads = nullptr;
  int32_t* nheads = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  const int64_t nk = max_slots > 0 ? max_slots : 1;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t group_warps = (int64_t)nsm * 8;
  const int64_t spw = 4 * (g.cap0 + kWaveMax + 64);  // u64 words per warp: cbuf, sbuf, ibuf, dbuf, pr
  chk(cudaMallocAsync((void**)&off_d, sizeof(int64_t) * off_h.size(), s));
  chk(cudaMallocAsync((void**)&keys, sizeof(uint64_t) * nk, s));
  chk(cudaMallocAsync((void**)&keys2, sizeof(uint64_t) * nk, s));
  chk(cudaMallocAsync((void**)&heads, sizeof(int64_t) * nk, s));
  chk(cudaMallocAsync((void**)&nheads, sizeof(int32_t), s));
  chk(cudaMallocAsync((void**)&scratch, sizeof(uint64_t) * group_warps * spw, s));
  if (e == cudaSuccess) chk(cub::DeviceRadixSort::SortKeys(nullptr, cub_bytes, keys, keys2, (int)nk, 0, 48, s));
  if (e == cudaSuccess) chk(cudaMallocAsync(&cub_tmp, cub_bytes, s));
  if (e == cudaSuccess)
    chk(cudaMemcpyAsync(off_d, off_h.data(), sizeof(int64_t) * off_h.size(), cudaMemcpyHostToDevice, s));
  const ILayout Ly = ilayout(efc);
  const int wpb = 4;
  const size_t ismem = (size_t)Ly.bytes * wpb;
  const size_t gsmem = (size_t)(4 * kCapMax * 2 + 64) * wpb;
  if (e == cudaSuccess)
    chk(cudaFuncSetAttribute(insert_kernel<LPR, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ismem));
  for (size_t w = 0; e == cudaSuccess && w + 1 < wave_lo.size(); ++w) {
    const int64_t p = wave_lo[w];
    const int32_t B = (int32_t)(wave_lo[w + 1] - p);
    const int64_t ns = off_h[off_at[w] + B];
    const int32_t blocks = (B + wpb - 1) / wpb;
    insert_kernel<LPR, CPL><<<blocks, wpb * 32, ismem, s>>>(g, p, B, wave_entry[w], wave_top[w], efc, sel0,
                                                            keep_pruned, off_d + off_at[w], keys);
    chk(cudaGetLastError());
    if (ns == 0) continue;
    chk(cub::DeviceRadixSort::SortKeys(cub_tmp, cub_bytes, keys, keys2, (int)ns, 0, 48, s));
    chk(cudaMemsetAsync(nheads, 0, sizeof(int32_t), s));
    heads_kernel<<<(unsigned)((ns + 255) / 256), 256, 0, s>>>(keys2, ns, heads, nheads);
    chk(cudaGetLastError());
    int64_t gb = (ns + wpb - 1) / wpb;
    if (gb > group_warps / wpb) gb = group_warps / wpb;
    group_kernel<LPR, CPL><<<(unsigned)gb, wpb * 32, gsmem, s>>>(g, p, keys2, ns, heads, nheads, keep_pruned,
                                                                 scratch, spw);
    chk(cudaGetLastError());
  }
  entry_max[0] = entry;
  entry_max[1] = top;
  if (cub_tmp) cudaFreeAsync(cub_tmp, s);
  cudaFreeAsync(off_d, s);
  cudaFreeAsync(keys, s);
  cudaFreeAsync(keys2, s);
  cudaFreeAsync(heads, s);
  cudaFreeAsync(nheads, s);
  cudaFreeAsync(scratch, s);
  return e;
}

}  // namespace

size_t build_smem_bytes(int32_t efc) { return (size_t)ilayout(efc).bytes * 4; }

cudaError_t build_graph_gpu(const uint8_t* codes, const int32_t* xnorm, int64_t n, int32_t d_pad32,
                            const int32_t* levels_d, const int32_t* levels_h, const int32_t* up_off_d, int32_t M,
                            int32_t efc, int32_t flags, int32_t batch_div, int32_t* adj0_d, int32_t* adj_up_d,
                            int32_t* entry_max, cudaStream_t s) {
  BView g;
  g.codes = codes;
  g.xnorm = xnorm;
  g.d_pad = d_pad32;
  g.M = M;
  g.cap0 = 2 * M;
  g.adj0 = adj0_d;
  g.adj_up = adj_up_d;
  g.up_off = up_off_d;
  g.levels = levels_d;
  const int32_t keep_pruned = flags & 1, sel0 = (flags & 2) ? 2 * M : M;
  if (batch_div <= 0) batch_div = 32;
  const Shape sh = shape_of(d_pad32);
#define AQR_RUN(L_, C_) \
  return run_waves<L_, C_>(g, n, levels_h, efc, sel0, keep_pruned, batch_div, entry_max, s)
  switch (sh.lpr * 10 + sh.cpl) {
    case 11: AQR_RUN(1, 1);
    case 21: AQR_RUN(2, 1);
    case 41: AQR_RUN(4, 1);
    case 81: AQR_RUN(8, 1);
    case 161: AQR_RUN(16, 1);
    case 321: AQR_RUN(32, 1);
    case 322: AQR_RUN(32, 2);
    default: return cudaErrorInvalidValue;
  }
#undef AQR_RUN
}

}  // namespace aqr
