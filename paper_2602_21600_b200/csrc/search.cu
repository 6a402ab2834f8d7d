// search.cu -- fused AQR-HNSW query search on sm_100a (aqr_search / aqr_rerank).
//
// One warp per query, persistent grid (atomic query counter), 24 warps per SM.  Per query,
// all inside the kernel (Alg2):
//   1. quantize the query (Alg2 l.4);
//   2. greedy descent through layers max_level..1 on d^q (R8);
//   3. layer-0 beam with ef on d^q (Alg2 l.6-7), "flag form" (R8): W is a sorted
//      list of <= ef 64-bit keys (d^q << 32 | id << 1 | expanded) in shared memory; each step
//      expands the smallest unexpanded entry: its adjacency row (requested during the previous
//      insert) -> its neighbours' code rows gathered with 256-bit loads (LPR lanes per row) ->
//      d^q = |q^|^2 + |x^|^2 - 2 q^.x^ with dp4a (|x^|^2 precomputed per node) -> filter
//      against max W -> dedupe + insertion point by binary search in W -> insert (per-segment
//      block moves); wide rows (d_pad > 512) are staged by TMA bulk copies instead;
//   4. Stage 2: decode + asymmetric fp32 distance for C = W[0:N_c] (Alg2 l.8-13);
//   5. early termination (Alg2 l.15-16, fp64 test on fp32 values, R11);
//   6. Stage 3: exact fp32 distance over the retained fp32 rows (Alg2 l.18-22, FMA P:197);
//   7. assembly + top-k (Alg2 l.23-24; fill reading R10 or union S:515) and the store.
// traversal = fp32 (template FP) is the paper's baseline HNSW on the same graph (R22).
//
// The path is a gather (pointer chasing), not a contraction: no tensor cores (north_star).
// Integer results (codes, d^q, W, visit order, ids) are bit-exact with the oracle; fp32
// sums use a lane-strided FMA order and agree with the oracle's sequential order within
// 1e-5 relative (north_star tolerance); the fp32 baseline uses the canonical order R(L) and
// is bit-exact.  Compile-time AQR_* knobs below record measured alternatives.
#include <cfloat>
#include <cstdio>
#include <climits>

#include "aqr_internal.cuh"

namespace aqr {

namespace {

// tuning knobs (compile-time; tools/perf.py A/B-tests variants built with -D overrides)
#ifndef AQR_WARPS_PER_CTA
#define AQR_WARPS_PER_CTA 4
#endif
#ifndef AQR_MIN_CTAS
#define AQR_MIN_CTAS 6  // 6 CTAs x 4 warps (<= 80 regs).  7 (<= 72 regs; the shared memory fits at C2
                        // ef 784 since NDA) measured 13.7 vs 10.2 ms: the register cap costs more
#endif
#ifndef AQR_NOCOMPACT
#define AQR_NOCOMPACT 1  // GATHER without the visited hash: score the adjacency row as stored
#endif
#ifndef AQR_SPEC2
#define AQR_SPEC2 0  // 1: row of the likely next expansion loaded early, its codes prefetched to L2
                     // (measured slower, 13.9 vs 12.8 ms, and no single-query latency gain)
#endif
#ifndef AQR_BALANCE
#define AQR_BALANCE 0  // 1: grid sized so every warp serves the same number of queries (measured
                       // slower, 13.3 vs 12.8 ms: the extra warps of a partial round still hide latency)
#endif
#ifndef AQR_L2HINT
#define AQR_L2HINT 0  // 1: L2 eviction hints (code rows evict-last, adjacency rows evict-first); measured
                      // slightly slower (13.0 vs 12.8 ms), the codes are already ~78% L2-resident
#endif
#ifndef AQR_SHORT_SEG
#define AQR_SHORT_SEG 0  // 1: one-chunk fast path for W segments of <= 32 entries (measured neutral)
#endif
#ifndef AQR_W_SLACK
#define AQR_W_SLACK 0  // >0: free W slots before the list so an insert may move the head left instead of the
                       // tail right (parity-tested; measured slower at C2: 15.2 vs 13.2 ms with 128)
#endif
#ifndef AQR_SEARCH4
#define AQR_SEARCH4 0  // 1: 4-ary W lower bound (three probes per step; measured slower at throughput)
#endif
#ifndef AQR_ROWS_PER_PASS
#define AQR_ROWS_PER_PASS 8  // 16-byte code chunks in flight per lane per gather pass (8: 4 rows of 32 B; 16 measured slower)
#endif
#ifndef AQR_LB_SHAR
#define AQR_LB_SHAR 1  // 1: W lower bound in Shar's form, probes unrolled (ef <= 16383)
#endif
#ifndef AQR_LB_FIXED
#define AQR_LB_FIXED 1  // 1: W lower bound with a warp-uniform trip count (no lane divergence)
#endif
#ifndef AQR_FASTDIV
#define AQR_FASTDIV 1  // 1: Stage 2 decode by reciprocal + one FMA correction (exact, checked at upload)
#endif
#ifndef AQR_PREFETCH_ROW
#define AQR_PREFETCH_ROW 1
#endif
#ifndef AQR_FINISH_NOINLINE
#define AQR_FINISH_NOINLINE 0  // 1: Stages 2-3 out of line (their registers stay out of the beam's allocation)
#endif
#ifndef AQR_HASH_DIRECT
#define AQR_HASH_DIRECT 1  // 1: the shared-memory visited set is direct-mapped (0: 8-probe open addressing)
#endif
#ifndef AQR_HASH_TAG16
#define AQR_HASH_TAG16 1  // 1: the direct-mapped visited set stores 16-bit tags of a bijective hash (half the bytes per slot)
#endif
#ifndef AQR_VBM_LOAD
#define AQR_VBM_LOAD 1  // 1: visited-bitmap test by an L2 load (ld.cg), the bit set by a fire-and-forget RED
                        // only for first visits (0: one atomicOr per neighbour, its old value the test).
                        // C4 ef 2480: 25.7 -> 23.9 ms; C1 ef 64 0.22 -> 0.236 ms (C1 benches the smem table)
#endif
#ifndef AQR_VBM_HINT
#define AQR_VBM_HINT 1  // 1: visited-bitmap atomics carry an L2 evict-last policy
#endif
#ifndef AQR_WIDE_U
#define AQR_WIDE_U 16  // > 0: wide-row kernels (LPR 32) read this many rows per pass, registers unbounded (0: 8, 80 regs)
#endif
#ifndef AQR_KNOWN_NEXT
#define AQR_KNOWN_NEXT 1  // 1: the next expansion's W position carried over (no pick scan)
#endif
#ifndef AQR_ADAPTIVE
#define AQR_ADAPTIVE 1  // 0: compile out the adaptive re-rank depth (A/B of its cost)
#endif
#ifndef AQR_MOVE32
#define AQR_MOVE32 3  // W segments move top first: 3 = 128 per step while long, then 64 (2 = 64 only, 1 = 32, 0 = 128)
#endif
#ifndef AQR_KW_HINT
#define AQR_KW_HINT 1024  // ef >= this: after a new key is expanded next, the first unexpanded entry
                          // after it is known from the insert (no scan over the expanded entries in
                          // between): C3 ef 5888 -4.3% (cooperative kernel); see AQR_KW_HINT_SINGLE (0: off)
#endif
#ifndef AQR_KW_HINT_SINGLE
#define AQR_KW_HINT_SINGLE 0  // 1: AQR_KW_HINT in the one-warp kernel too
#endif
#ifndef AQR_FLAT_MERGE
#define AQR_FLAT_MERGE 10  // > 0: the W insert takes one chunked pass when np * this > entries moved (0: off;
                          // 10: C5 2.98 -> 2.86 ms, C2 9.64 -> 9.60; 40: C2 9.92)
#endif
#ifndef AQR_PF_PASSES
#define AQR_PF_PASSES 0  // 1: before the first gather pass of an expansion, the code rows of the later
                         // passes are prefetched into L2 (prefetch.global.L2: no registers, no result)
#endif
#ifndef AQR_PF_ROW
#define AQR_PF_ROW 0  // 1: the scan for the first unexpanded W entry after the pick runs before the scoring, and
                      // that node's adjacency row (the next expansion unless a smaller new key arrives) is
                      // prefetched into L2
#endif
#ifndef AQR_PF_FINISH
#define AQR_PF_FINISH 0  // 1: Stage 2's code rows and Stage 3's fp32 rows are prefetched into L2 before their
                         // 4-row loops (each loop step is otherwise one exposed round trip)
#endif
#ifndef AQR_CMIN_GUARD
#define AQR_CMIN_GUARD 0  // 1: the warp-wide minimum of the new keys is skipped when the expansion has none
#endif
#ifndef AQR_HASH_2WAY
#define AQR_HASH_2WAY 1  // 1: the 16-bit-tag visited table is two-way set associative (LRU) in the same bytes
                         // (C5 shard 2^10 slots 2.96 -> 2.79 ms, 2^11 3.39 -> 2.96, C1 2^13 0.215 -> 0.213); 2: four-way
#endif
#ifndef AQR_FUSED_FILTER
#define AQR_FUSED_FILTER 1  // 1: layer-0 scoring and the max-W filter in one pass (list_filter)
#endif

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kEmpty = 0xffffffffu;

// AQR_CHECKS=1 (a test build, libaqr_checked.so): bounds checks on every shared-memory array
// index and every gathered node id; a violation prints its line and traps.  compute-sanitizer is
// closed on this pool, so the GPU suite runs against this build instead (tools/gpu/checked.sh)
#ifndef AQR_CHECKS
#define AQR_CHECKS 0
#endif
#if AQR_CHECKS
#define AQR_ASSERT(cond)                                                                     \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      printf("AQR_CHECKS: %s failed at search.cu:%d (block %d thread %d)\n", #cond, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                            \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)
#else
#define AQR_ASSERT(cond) \
  do {                   \
  } while (0)
#endif
constexpr int kProbes = 8;

// ------------------------------------------------------------------------------------
// small helpers
// ------------------------------------------------------------------------------------
// %globaltimer: the GPU's nanosecond wall clock (per-query latency, aqr_debug.t_ns)
__device__ __forceinline__ int64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (int64_t)t;
}

__device__ __forceinline__ uint64_t qkey(uint32_t d, int32_t id) {
  return ((uint64_t)d << 32) | ((uint64_t)(uint32_t)id << 1);
}
__device__ __forceinline__ int32_t qkey_id(uint64_t k) { return (int32_t)((uint32_t)k >> 1); }
__device__ __forceinline__ uint32_t qkey_d(uint64_t k) { return (uint32_t)(k >> 32); }

__device__ __forceinline__ uint32_t fkey(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}
__device__ __forceinline__ uint64_t akey(float d, int32_t id) {
  return ((uint64_t)fkey(d) << 32) | (uint32_t)id;
}

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(kFull, (uint32_t)v, m), hi = __shfl_xor_sync(kFull, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  uint32_t lo = __shfl_sync(kFull, (uint32_t)v, src), hi = __shfl_sync(kFull, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
// warp-wide 64-bit minimum: two redux.sync (REDUX) on the high then the low word
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  const uint32_t hi = (uint32_t)(v >> 32);
  const uint32_t mh = __reduce_min_sync(kFull, hi);
  const uint32_t ml = __reduce_min_sync(kFull, hi == mh ? (uint32_t)v : 0xffffffffu);
  return ((uint64_t)mh << 32) | ml;
}

// ---- mbarrier + bulk (TMA) copy helpers (sm_90+ PTX; UBLKCP in SASS) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// arrive (count 1) and announce `bytes` of transaction, then copy `bytes` global -> shared
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// number of W keys strictly less than key, ignoring the expanded flag bit
// (key has flag 0 and keys differ above bit 0, so a[i] < key needs no mask.)  4-ary search: three
// independent probes per step halve the dependent shared-load chain of a binary search.
__device__ __forceinline__ int lower_bound_w(const uint64_t* a, int n, uint64_t key) {
#if AQR_SEARCH4
  int lo = 0, len = n;  // the answer lies in [lo, lo + len]
  while (len >= 4) {
    const int p1 = lo + (len >> 2), p2 = lo + (len >> 1), p3 = lo + ((3 * len) >> 2);
    const uint64_t v1 = a[p1], v2 = a[p2], v3 = a[p3];
    const int hi = lo + len;
    if (v3 < key) {
      lo = p3 + 1;
      len = hi - lo;
    } else if (v2 < key) {
      lo = p2 + 1;
      len = p3 - lo;
    } else if (v1 < key) {
      lo = p1 + 1;
      len = p2 - lo;
    } else {
      len = p1 - lo;
    }
  }
  int hi = lo + len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
#elif AQR_LB_SHAR
  // Shar's form: after the first probe the window [i, i + k] lies inside [0, n], so the remaining
  // probes need no bound check; they are unrolled by a switch on log2(k) (warp-uniform: n is the
  // list size), each one LDS.64 at a constant offset from a[i] plus a 64-bit compare and add
  if (n <= 0) return 0;
  const int lg = 31 - __clz(n);
  const int k = 1 << lg;
  int i = a[k - 1] < key ? n - k : 0;
  switch (lg) {
#define AQR_LB_STEP(L) \
  case L:              \
    if (a[i + (1 << ((L)-1)) - 1] < key) i += 1 << ((L)-1);
    AQR_LB_STEP(13) AQR_LB_STEP(12) AQR_LB_STEP(11) AQR_LB_STEP(10) AQR_LB_STEP(9) AQR_LB_STEP(8) AQR_LB_STEP(7)
    AQR_LB_STEP(6) AQR_LB_STEP(5) AQR_LB_STEP(4) AQR_LB_STEP(3) AQR_LB_STEP(2) AQR_LB_STEP(1)
#undef AQR_LB_STEP
    default:
      break;
  }
  // the probes decide min(lb - i, k - 1); one more settles lb - i = k (a[i] is in range)
  if (a[i] < key) ++i;
  return i;
#elif AQR_LB_FIXED
  // greedy bit-by-bit: the answer's bits from bit_floor(n) down; the trip count depends only on
  // the warp-uniform n, so the lanes of a warp never diverge
  int lo = 0;
  for (int step = n > 0 ? 1 << (31 - __clz(n)) : 0; step > 0; step >>= 1)
    if (lo + step <= n && a[lo + step - 1] < key) lo += step;
  return lo;
#else
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
#endif
}

// ------------------------------------------------------------------------------------
// per-warp shared-memory layout
// ------------------------------------------------------------------------------------
constexpr int kStage = 8;  // rows per stage buffer of the staged (TMA) wide-row gather

struct Layout {
  // runtime part of the per-warp layout; the hot arrays of the beam (Hot<> below) sit at
  // compile-time offsets before W, so every access to them is [warp base + immediate]
  int o_w, o_qc, o_qf, o_h, o_s23, per_warp;
  int o_stg;      // staged wide-row gather: its 2 x kStage row buffer (after the visited hash)
  int q_alias;    // 1: query codes / fp32 query live in the hot arrays (rebuilt for Stage 2)
  int region;     // bytes of the hash / block-buffer region (reused by Stage 2/3)
  int buf_bytes;  // INLINE: one staged block (128-byte aligned)
};

__host__ __device__ constexpr int al16(int x) { return (x + 15) & ~15; }

// rows per lane per list_dists pass: AQR_ROWS_PER_PASS 16-byte chunks in flight per lane
template <int CPL, int LPR = 0>
__host__ __device__ constexpr int rows_u() {
  // wide rows (LPR 32: one row per warp step): AQR_WIDE_U rows per pass, with the register
  // budget of a few resident warps (see the launch bounds of search_kernel)
  return (LPR == 32 && AQR_WIDE_U > 0) ? AQR_WIDE_U / CPL
         : (AQR_ROWS_PER_PASS / (2 * CPL) < 4 ? 4 : AQR_ROWS_PER_PASS / (2 * CPL) / 4 * 4);
}

// per-query counters + mbarriers at the end of the hot region: live for the whole kernel, so a
// query aliased into the hot region (make_layout) stops short of them
constexpr int kHotTail = 80;

// the beam's per-warp scratch for adjacency rows of up to CAP entries (CAP = 56 or 160).
// NDA (the fused list_filter path): the beam never stores d^q, so the greedy descent's d^q
// array borrows cs and the merge's sorted insertion points (slb) borrow nb -- 4 CAP bytes less
// per warp
template <int LPR, int CPL, int CAP, bool NDA = false>
struct Hot {
  static constexpr int PASS = (32 / LPR) * rows_u<CPL, LPR>();  // rows read per list_dists pass
  static constexpr int NB1 = (CAP + PASS - 1) / PASS * PASS;
  static constexpr int NB = NB1 > (CAP + 31) / 32 * 32 ? NB1 : (CAP + 31) / 32 * 32;
  static constexpr int o_nb = 0;                                  // int32 [NB] neighbour ids
  static constexpr int o_cand = o_nb + al16(4 * NB) + (NDA ? 0 : al16(4 * CAP));  // u64 [CAP] new W keys
  static constexpr int o_cs = o_cand + 8 * CAP;                   // u64 [CAP] survivors / sorted keys
  static constexpr int o_nd = NDA ? o_cs : o_nb + al16(4 * NB);   // int32 [CAP] d^q
  static constexpr int o_slb = NDA ? o_nb : o_nd;                 // int32 [CAP] sorted insertion points
  static constexpr int o_lb = o_cs + 8 * CAP;                     // int32 [CAP] W lower bounds
  static constexpr int o_cnt = o_lb + al16(4 * CAP);              // int32 [16] per-query counters (debug)
  static constexpr int o_bar = o_cnt + 64;                        // mbarriers (INLINE / staged)
  static constexpr int bytes = o_bar + 16;                        // W follows
  static_assert(bytes - o_cnt == kHotTail, "hot tail");
};

// the Hot<> variant a kernel instantiation uses
template <int LPR, bool INL, bool FP>
__host__ __device__ constexpr bool nd_alias() {
  return !INL && !FP && AQR_FUSED_FILTER && LPR < 32;
}

// the visited hash's slot format for this index (see visit_new16): 16-bit tags when the id range
// [0, 2^B), 2^B >= n, splits into hbits slot bits and at most 15 tag bits, else 32-bit ids
void hash_params(const IndexView& ix, SearchCfg& c) {
  c.htag = -1;
  c.hmul = c.hmaskb = 0u;
  if (!AQR_HASH_TAG16 || !AQR_HASH_DIRECT || c.hbits <= 0) return;
  int b = 0;
  while (b < 31 && ((int64_t)1 << b) < ix.n) ++b;
  if (b < c.hbits) b = c.hbits;
  if (b - c.hbits > 15) return;
  c.htag = b - c.hbits;
  c.hmaskb = b >= 32 ? ~0u : ((1u << b) - 1u);
  c.hmul = (uint32_t)(2654435769ull >> (32 - b)) | 1u;  // ~2^b / golden ratio, odd
}

Layout make_layout(const IndexView& ix, const SearchCfg& c, int hot_bytes) {
  Layout L;
  int o = hot_bytes;
  L.o_w = o; o += al16(8 * (c.ef + 1 + AQR_W_SLACK));
  // the query (codes + fp32) is only read before the beam and in Stage 2/3: when it fits it
  // borrows the beam's scratch (AQR traversal; the fp32 baseline reads it throughout)
  const int qbytes = al16(4 * ix.d4) + al16(ix.d_pad);
  L.buf_bytes = (ix.blk_bytes + 127) & ~127;
  // INLINE block buffer (AQR traversal on an INLINE index), else the visited hash.  The FP32
  // traversal runs the GATHER kernel even on an INLINE index, so it needs the hash region
  const int hbytes = c.hbits > 0 ? ((c.htag >= 0 ? 2 : 4) << c.hbits) : 0;
  L.region = (ix.blk && !c.fp32) ? L.buf_bytes : hbytes;
  int stg_rel = 0;
  if (c.staged) {  // staged_dists: 2 x kStage wide rows, after the visited hash (both live in the beam)
    stg_rel = (hbytes + 127) & ~127;
    const int st = stg_rel + 2 * kStage * ix.d_pad;
    if (st > L.region) L.region = st;
  }
  // ... or the staged gather's buffer (wide rows: the query is too big for the hot arrays)
  // (the counters and mbarriers at the end of the hot region stay live: the query stops short)
  const bool in_hot = !c.fp32 && qbytes <= hot_bytes - kHotTail;
  const bool in_stage = !c.fp32 && !in_hot && c.staged && !ix.blk && c.hbits == 0 && qbytes <= L.region;
  L.q_alias = in_hot || in_stage;
  if (!L.q_alias) {
    L.o_qc = o; o += al16(ix.d_pad);
    L.o_qf = o; o += al16(4 * ix.d4);
  }
  o = (o + 127) & ~127;
  L.o_h = o; o += al16(L.region);
  L.o_stg = L.o_h + stg_rel;
  if (in_hot) {
    L.o_qf = 0;
    L.o_qc = al16(4 * ix.d4);
  } else if (in_stage) {
    L.o_qf = L.o_h;
    L.o_qc = L.o_h + al16(4 * ix.d4);
  }
  L.o_s23 = o; o += c.ef >= 2 * c.n_coarse ? 0 : al16(8 * c.n_coarse);
  L.per_warp = (o + 127) & ~127;
  return L;
}

// ------------------------------------------------------------------------------------
// Transpose reduction of U per-lane partial sums over groups of LPR lanes (LPR, U powers of 2).
// Step with offset o (o = LPR/2 .. 1) halves the live partials: lanes with (sub & o) keep the
// upper half of their rows, the others the lower half, each adding its partner's copy.  At the
// end (U >= LPR) lane `sub` holds, in part[0 .. U/LPR), the totals of rows sub*(U/LPR) + v.
// If U < LPR the last log2(LPR/U) steps are plain butterflies on a single value.
// ------------------------------------------------------------------------------------
template <int LPR, int U>
__device__ __forceinline__ void reduce_rows(int (&part)[U], int sub) {
  int n = U;  // live partials
#pragma unroll
  for (int o = LPR / 2; o >= 1; o >>= 1) {
    if (n > 1) {
      const int h = n / 2;
      const bool upper = (sub & o) != 0;
#pragma unroll
      for (int v = 0; v < U / 2; ++v) {
        if (v < h) {
          const int send = upper ? part[v] : part[v + h];
          const int keep = upper ? part[v + h] : part[v];
          part[v] = keep + __shfl_xor_sync(kFull, send, o);
        }
      }
      n = h;
    } else {
      part[0] += __shfl_xor_sync(kFull, part[0], o);
    }
  }
}

// ------------------------------------------------------------------------------------
// d^q for a list of node ids: LPR lanes per code row, CPL 32-byte chunks per lane (one
// LDG.256 each; code rows are padded to a multiple of 32 bytes at upload)
// d^q = sum q^2 + sum x^2 - 2 sum q x  (exact int32; dp4a on u8x4 words)
// ------------------------------------------------------------------------------------
struct C32 {
  uint4 a, b;
};

__device__ __forceinline__ void ldg256(const void* p, C32& v) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.a.x), "=r"(v.a.y), "=r"(v.a.z), "=r"(v.a.w), "=r"(v.b.x), "=r"(v.b.y), "=r"(v.b.z),
                 "=r"(v.b.w)
               : "l"(p));
}

// the same with an L2 evict-last hint (LDG.E.NA.ELL2.256): the code rows are the data reused
// across queries, so they should outlive the adjacency rows and fp32 rows in L2
__device__ __forceinline__ void ldg256_keep(const void* p, C32& v) {
#if AQR_L2HINT
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.a.x), "=r"(v.a.y), "=r"(v.a.z), "=r"(v.a.w), "=r"(v.b.x), "=r"(v.b.y), "=r"(v.b.z),
                 "=r"(v.b.w)
               : "l"(p));
#else
  ldg256(p, v);
#endif
}

// scalar loads with an L2 eviction policy (createpolicy + L2::cache_hint)
__device__ __forceinline__ int32_t ldg_first(const int32_t* p) {
#if AQR_L2HINT
  uint64_t pol;
  int32_t v;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ int32_t ldg_last(const int32_t* p) {
#if AQR_L2HINT
  uint64_t pol;
  int32_t v;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ void dp4a_c32(const C32& w, const C32& q, unsigned& xx, unsigned& qx) {
  xx = __dp4a(w.a.x, w.a.x, xx); qx = __dp4a(q.a.x, w.a.x, qx);
  xx = __dp4a(w.a.y, w.a.y, xx); qx = __dp4a(q.a.y, w.a.y, qx);
  xx = __dp4a(w.a.z, w.a.z, xx); qx = __dp4a(q.a.z, w.a.z, qx);
  xx = __dp4a(w.a.w, w.a.w, xx); qx = __dp4a(q.a.w, w.a.w, qx);
  xx = __dp4a(w.b.x, w.b.x, xx); qx = __dp4a(q.b.x, w.b.x, qx);
  xx = __dp4a(w.b.y, w.b.y, xx); qx = __dp4a(q.b.y, w.b.y, qx);
  xx = __dp4a(w.b.z, w.b.z, xx); qx = __dp4a(q.b.z, w.b.z, qx);
  xx = __dp4a(w.b.w, w.b.w, xx); qx = __dp4a(q.b.w, w.b.w, qx);
}

__device__ __forceinline__ void dp4a_qx(const C32& w, const C32& q, unsigned& qx) {
  qx = __dp4a(q.a.x, w.a.x, qx);
  qx = __dp4a(q.a.y, w.a.y, qx);
  qx = __dp4a(q.a.z, w.a.z, qx);
  qx = __dp4a(q.a.w, w.a.w, qx);
  qx = __dp4a(q.b.x, w.b.x, qx);
  qx = __dp4a(q.b.y, w.b.y, qx);
  qx = __dp4a(q.b.z, w.b.z, qx);
  qx = __dp4a(q.b.w, w.b.w, qx);
}


// after reduce_rows, write the row totals r0 + g U + u held by this lane
template <int LPR, int U>
__device__ __forceinline__ void store_rows(const int (&part)[U], int r0, int g, int sub, int m, int qq, int32_t* out) {
  constexpr int PER = U >= LPR ? U / LPR : 1;
  constexpr int REP = U >= LPR ? 1 : LPR / U;
#pragma unroll
  for (int v = 0; v < PER; ++v) {
    const int u = U >= LPR ? sub * PER + v : sub / REP;
    const int r = r0 + g * U + u;
    if ((sub % REP) == 0 && r < m) out[r] = qq + part[v];
  }
}

template <int LPR, int CPL, int UU = 0>
__device__ __forceinline__ void list_dists(const IndexView& ix, const C32 (&qreg)[CPL], int qq,
                                           const int32_t* ids, int m, int32_t* out, int lane) {
  constexpr int G = 32 / LPR;
  // all loads of a pass are issued before any is consumed: U rows per lane, G * U rows per pass,
  // so a typical layer-0 expansion (<= 64 rows of 128 B) costs ONE DRAM round trip
  constexpr int U = UU > 0 ? UU : rows_u<CPL, LPR>();
  static_assert(U % 4 == 0, "U must be a multiple of 4");
  const int g = lane / LPR, sub = lane % LPR;
  const int nch = ix.d_pad >> 5;
  for (int r0 = 0; r0 < m; r0 += G * U) {
    // lane group g owns the U consecutive rows r0 + g U + u: their ids come in U/4 16-byte
    // shared loads (ids is padded to a whole pass, see make_layout)
    int idv[U];
#pragma unroll
    for (int u4 = 0; u4 < U; u4 += 4) {
      const int4 t4 = *reinterpret_cast<const int4*>(ids + r0 + g * U + u4);
      idv[u4] = t4.x;
      idv[u4 + 1] = t4.y;
      idv[u4 + 2] = t4.z;
      idv[u4 + 3] = t4.w;
    }
    // |x^|^2 (precomputed per node) of the rows whose totals this lane holds after the reduction;
    // d^q = |q^|^2 + |x^|^2 - 2 q^.x^ then needs dp4a only for q^.x^
    constexpr int PER = U >= LPR ? U / LPR : 1;
    constexpr int REP = U >= LPR ? 1 : LPR / U;
    int xn[PER];
#pragma unroll
    for (int v = 0; v < PER; ++v) {
      const int u = U >= LPR ? sub * PER + v : sub / REP;
      const int r = r0 + g * U + u;
      const int id = r < m ? ids[r] : -1;
      xn[v] = id >= 0 ? ldg_last(ix.xnorm + id) : 0;
    }
    C32 buf[U][CPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + g * U + u;
      const int id = r < m ? idv[u] : -1;
      AQR_ASSERT(id < ix.n);
      const uint8_t* row = ix.codes + (int64_t)(id < 0 ? 0 : id) * ix.d_pad;
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = sub + LPR * t;
        if (id >= 0 && c < nch) {
          ldg256_keep(row + 32 * c, buf[u][t]);
        } else {
          buf[u][t].a = make_uint4(0, 0, 0, 0);
          buf[u][t].b = make_uint4(0, 0, 0, 0);
        }
      }
    }
    int part[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      unsigned qx = 0;
#pragma unroll
      for (int t = 0; t < CPL; ++t) dp4a_qx(buf[u][t], qreg[t], qx);
      part[u] = -2 * (int)qx;
    }
    // transpose-reduce across the LPR lanes of a row group (U/2 + U/4 + ... shuffles instead of
    // U * log2(LPR)); afterwards lane `sub` holds the total of row u = sub * PER + v in part[v]
    // (U >= LPR), or, when U < LPR, every lane holds the total of row sub / (LPR / U)
    reduce_rows<LPR, U>(part, sub);
#pragma unroll
    for (int v = 0; v < PER; ++v) part[v] += xn[v];
    store_rows<LPR, U>(part, r0, g, sub, m, qq, out);
  }
}

// ------------------------------------------------------------------------------------
// The layer-0 expansion's scoring and filter in one pass (AQR_FUSED_FILTER): d^q of every
// neighbour as list_dists computes it, but instead of storing d^q and re-reading it for the
// filter, the lane that holds a row's total forms its W key and tests it against max W at once;
// the survivors (key < maxk, Alg2 l.7's bounded beam) are compacted into cs.  Returns their count.
// Requirements: ids[0 .. round_up(m, pass)) readable, entries past the row's end = -1 (the
// callers pad nb), so no row needs an `r < m` guard.  An absent row (-1) reads a stand-in row and
// is dropped by the `id >= 0` test; a lane whose chunk lies past the row's end re-reads the last
// chunk, multiplied by the query's zero chunk.  Same integers as list_dists.
// ------------------------------------------------------------------------------------
template <int LPR, int CPL, int UU = 0>
__device__ __forceinline__ int list_filter(const IndexView& ix, const C32 (&qreg)[CPL], int qq,
                                           const int32_t* ids, int m, const uint64_t* W, int size, int ef,
                                           uint64_t* cs, int lane) {
  constexpr int G = 32 / LPR;
  constexpr int U = UU > 0 ? UU : rows_u<CPL, LPR>();
  constexpr int PER = U >= LPR ? U / LPR : 1;
  constexpr int REP = U >= LPR ? 1 : LPR / U;
  const int g = lane / LPR, sub = lane % LPR;
  const int nch = ix.d_pad >> 5;
  const uint32_t dpad = (uint32_t)ix.d_pad;
  // stand-in for absent rows: the list's first neighbour (an L2-hot row that differs from warp to
  // warp; a fixed row would put every warp's absent rows on one L2 line -- measured, a hot spot)
  const int alt = max(ids[0], 0);
  int np0 = 0;
#if AQR_PF_PASSES
  // a pass waits for the slowest of its G * U rows (some row misses L2 in nearly every pass): the
  // rows of passes 2.. are requested now, so those passes find them in L2
  for (int i = G * U + lane; i < m; i += 32) {
    const int id = ids[i];
    if (id >= 0) {
      // every 128-byte line the row touches (rows of d_pad = 96 straddle lines)
      const uint64_t a0 = reinterpret_cast<uint64_t>(ix.codes) + (uint64_t)(uint32_t)id * dpad;
      for (uint64_t a = a0 & ~127ull; a < a0 + dpad; a += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
#if AQR_PF_PASSES >= 2
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ix.xnorm + id));
#endif
    }
  }
#endif
  for (int r0 = 0; r0 < m; r0 += G * U) {
    const int32_t* idp = ids + r0 + g * U;
    // |x^|^2 of the rows whose totals this lane holds after the reduction
    int xn[PER];
#pragma unroll
    for (int v = 0; v < PER; ++v) {
      const int id = idp[U >= LPR ? sub * PER + v : sub / REP];
      xn[v] = id >= 0 ? __ldg(ix.xnorm + id) : 0;
    }
    // an absent row (-1) reads the stand-in row `alt` instead (no predicate, no zero fill); its
    // total is dropped by the id test below
    C32 buf[U][CPL];
#pragma unroll
    for (int u4 = 0; u4 < U; u4 += 4) {
      const int4 t4 = *reinterpret_cast<const int4*>(idp + u4);
      const int idv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        AQR_ASSERT(idv[e] < ix.n && alt < ix.n);
        const uint8_t* row = ix.codes + (uint64_t)(uint32_t)(idv[e] >= 0 ? idv[e] : alt) * dpad;
#pragma unroll
        for (int t = 0; t < CPL; ++t) ldg256_keep(row + 32 * min(sub + LPR * t, nch - 1), buf[u4 + e][t]);
      }
    }
    int part[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      unsigned qx = 0;
#pragma unroll
      for (int t = 0; t < CPL; ++t) dp4a_qx(buf[u][t], qreg[t], qx);
      part[u] = -2 * (int)qx;
    }
    reduce_rows<LPR, U>(part, sub);
    // the filter against max W (W is not modified during the pass)
    const uint64_t maxk = size >= ef ? (W[size - 1] & ~1ull) : ~0ull;
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int v = 0; v < PER; ++v) {
      const int id = idp[U >= LPR ? sub * PER + v : sub / REP];
      const uint64_t kk = ((uint64_t)(uint32_t)(qq + part[v] + xn[v]) << 32) | ((uint64_t)(uint32_t)id << 1);
      const bool ok = (REP == 1 || (sub % REP) == 0) && id >= 0 && kk < maxk;
      const uint32_t mk = __ballot_sync(kFull, ok);
      AQR_ASSERT(!ok || np0 + __popc(mk & lt) < m + 32);
      if (ok) cs[np0 + __popc(mk & lt)] = kk;
      np0 += __popc(mk);
    }
  }
  return np0;
}

// ------------------------------------------------------------------------------------
// d^q for wide code rows (d_pad > 512, LPR = 32: one row per warp step, e.g. C4 d = 960): a
// register pass holds only U = 8 rows, so a 140-neighbour expansion would take ~18 dependent
// round trips.  Instead the rows are bulk-copied (cp.async.bulk, TMA) into a double-buffered
// shared stage of kStage rows each, the copies of chunk i+1 in flight while chunk i is scored:
// about one round trip per expansion.  Same arithmetic as list_dists (exact int32 d^q).
// ------------------------------------------------------------------------------------
template <int CPL>
__device__ __forceinline__ void staged_dists(const IndexView& ix, const C32 (&qreg)[CPL], int qq, const int32_t* ids,
                                             int m, int32_t* out, int lane, uint8_t* stage, uint64_t* bars,
                                             uint32_t& ph) {
  constexpr int LPR = 32, U = kStage;
  const int nch = ix.d_pad >> 5;
  const int nck = (m + U - 1) / U;
  auto issue = [&](int ck) {
    const int b = ck & 1, r0 = ck * U;
    const int id = (lane < U && r0 + lane < m) ? ids[r0 + lane] : -1;
    const int nv = __popc(__ballot_sync(kFull, id >= 0));
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bars + b)),
                   "r"((uint32_t)(nv * ix.d_pad))
                   : "memory");
    }
    __syncwarp();
    if (id >= 0) {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(stage + (size_t)(b * U + lane) * ix.d_pad)),
          "l"(ix.codes + (int64_t)id * ix.d_pad), "r"((uint32_t)ix.d_pad), "r"(smem_u32(bars + b))
          : "memory");
    }
  };
  if (nck > 0) issue(0);
  for (int ck = 0; ck < nck; ++ck) {
    if (ck + 1 < nck) issue(ck + 1);
    const int b = ck & 1, r0 = ck * U;
    // |x^|^2 of the row this lane will hold (REP = LPR / U lanes per row)
    constexpr int REP = LPR / U;
    const int ur = lane / REP;
    const int idr = r0 + ur < m ? ids[r0 + ur] : -1;
    const int xn = idr >= 0 ? __ldg(ix.xnorm + idr) : 0;
    mbar_wait(bars + b, (ph >> b) & 1u);
    ph ^= 1u << b;
    int part[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      unsigned qx = 0;
      const int r = r0 + u;
      const uint4* row = reinterpret_cast<const uint4*>(stage + (size_t)(b * U + u) * ix.d_pad);
      if (r < m && ids[r] >= 0) {
#pragma unroll
        for (int t = 0; t < CPL; ++t) {
          const int c = lane + LPR * t;
          if (c < nch) {
            C32 w;
            w.a = row[2 * c];
            w.b = row[2 * c + 1];
            dp4a_qx(w, qreg[t], qx);
          }
        }
      }
      part[u] = -2 * (int)qx;
    }
    reduce_rows<LPR, U>(part, lane);
    if ((lane % REP) == 0 && r0 + ur < m) out[r0 + ur] = qq + part[0] + xn;
    __syncwarp();  // the stage buffer is read before it is refilled
  }
}

// ------------------------------------------------------------------------------------
// FP32 baseline traversal (AQR_TRAVERSAL_FP32): exact distances of the query (fp32, shared
// memory) to a list of base rows (fp32, d4 = round_up(d, 8) floats).  LPR lanes per row, lane
// `sub` owns the 32-byte chunks c = sub + LPR t (one LDG.256 each); canonical order R(LPR):
// each lane accumulates its chunks in increasing c with one FMA per element, then a butterfly
// over the LPR lanes (offsets LPR/2 .. 1).  The key written is the order-preserving uint32 of
// the distance (fkey), so W and its (key, id) order are shared with the quantized path.
// ------------------------------------------------------------------------------------
template <int LPR>
__device__ __forceinline__ void fp_dists(const IndexView& ix, const float* qf, const int32_t* ids, int m,
                                         int32_t* out, int lane) {
  constexpr int G = 32 / LPR;
  constexpr int U = 4;  // rows per lane per pass (32 B each; half the AQR pass: the query chunk and
                        // the fp32 partial sums need the registers); nb is padded for 8
  const int g = lane / LPR, sub = lane % LPR;
  const int nchf = ix.d4 >> 3;
  for (int r0 = 0; r0 < m; r0 += G * U) {
    int idv[U];
#pragma unroll
    for (int u4 = 0; u4 < U; u4 += 4) {
      const int4 t4 = *reinterpret_cast<const int4*>(ids + r0 + g * U + u4);
      idv[u4] = t4.x;
      idv[u4 + 1] = t4.y;
      idv[u4 + 2] = t4.z;
      idv[u4 + 3] = t4.w;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + g * U + u >= m) idv[u] = -1;
    float part[U];
#pragma unroll
    for (int u = 0; u < U; ++u) part[u] = 0.0f;
    for (int c = sub; c < nchf; c += LPR) {
      C32 buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (idv[u] >= 0) {
          ldg256(ix.base + (int64_t)idv[u] * ix.d4 + 8 * c, buf[u]);
        } else {
          buf[u].a = make_uint4(0, 0, 0, 0);
          buf[u].b = make_uint4(0, 0, 0, 0);
        }
      }
      const float4 qa = reinterpret_cast<const float4*>(qf)[2 * c];
      const float4 qb = reinterpret_cast<const float4*>(qf)[2 * c + 1];
      const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t xw[8] = {buf[u].a.x, buf[u].a.y, buf[u].a.z, buf[u].a.w,
                                buf[u].b.x, buf[u].b.y, buf[u].b.z, buf[u].b.w};
        float acc = part[u];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xv = __uint_as_float(xw[e]);
          if (ix.metric == 0) {
            const float df = __fsub_rn(qv[e], xv);
            acc = __fmaf_rn(df, df, acc);
          } else {
            acc = __fmaf_rn(qv[e], xv, acc);
          }
        }
        part[u] = acc;
      }
    }
#pragma unroll
    for (int off = LPR / 2; off >= 1; off >>= 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) part[u] = __fadd_rn(part[u], __shfl_xor_sync(kFull, part[u], off));
    }
    if (sub == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + g * U + u;
        if (r < m) out[r] = (int32_t)fkey(ix.metric == 0 ? part[u] : __fsub_rn(1.0f, part[u]));
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// visited set: open-addressing hash of node ids in shared memory.  A full probe window
// reports "not visited" and overwrites the window's last slot (so the table keeps the most
// recently seen ids): a false negative only causes a re-evaluation, which the W dedupe
// absorbs (R15).  False positives cannot occur: a slot only ever holds
// an id that was inserted, and a hit requires the exact id.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ bool visit_new(uint32_t* h, int hbits, int32_t u, int& fails) {
#if AQR_HASH_DIRECT
  // direct-mapped: one slot per id hash, no probing, no atomics (the warp owns its table; two
  // lanes racing for a slot both report "new" and one id stays -- never a false positive)
  const uint32_t s0 = ((uint32_t)u * 2654435761u) >> (32 - hbits);
  if (h[s0] == (uint32_t)u) return false;
  h[s0] = (uint32_t)u;
  return true;
#endif
  const uint32_t hmask = (1u << hbits) - 1u;
  uint32_t s = ((uint32_t)u * 2654435761u) >> (32 - hbits);
#pragma unroll 1
  for (int p = 0; p < kProbes; ++p) {
    uint32_t old = atomicCAS(h + s, kEmpty, (uint32_t)u);
    if (old == kEmpty) return true;
    if (old == (uint32_t)u) return false;
    if (p + 1 < kProbes) s = (s + 1) & hmask;
  }
  // probe window full: overwrite its last slot (the table keeps the most recent ids)
  atomicExch(h + s, (uint32_t)u);
  ++fails;
  return true;
}

// direct-mapped visited set with 16-bit tags: x = (u * A) mod 2^B (A odd, 2^B >= n) is a bijection
// on [0, 2^B); its top hbits bits pick the slot and the low htag (<= 15) bits are stored, so (slot,
// tag) identifies u exactly -- a hit is never a false positive -- at half the bytes of an id slot
// (twice the slots in the same shared memory).  Empty slots hold 0xFFFF (no tag reaches 2^15)
// TW: the set-associative forms below (AQR_HASH_2WAY) are compiled only into the wide-row
// instantiations (CAP > 56: the configs that use the table, C1 / C5); compiled into the CAP 56
// kernel too, the unused code cost C2 0.4% (9.647 vs 9.605 ms, 3 x 6 runs each)
template <bool TW>
__device__ __forceinline__ bool visit_new16(uint16_t* h, const SearchCfg& c, int32_t u) {
  const uint32_t x = ((uint32_t)u * c.hmul) & c.hmaskb;
#if AQR_HASH_2WAY == 2
  // four-way sets (one 64-bit word, tags in LRU order from the low half of .x), tag = htag + 2 bits
  if (TW && c.htag < 14) {
    uint2* h64 = reinterpret_cast<uint2*>(h) + (x >> (c.htag + 2));
    const uint32_t t = x & ((4u << c.htag) - 1u);
    const uint2 w = *h64;
    const uint32_t t0 = w.x & 0xffffu, t1 = w.x >> 16, t2 = w.y & 0xffffu, t3 = w.y >> 16;
    if (t0 == t) return false;
    const bool hit = (t1 == t) | (t2 == t) | (t3 == t);
    // move to front; a hit on the last way or a miss drops t3
    const uint32_t ny = t1 == t ? w.y : (t2 == t ? ((t3 << 16) | t1) : ((t2 << 16) | t1));
    *h64 = make_uint2((t0 << 16) | t, ny);
    return !hit;
  }
#endif
#if AQR_HASH_2WAY
  // two-way sets in the same bytes: a set is one 32-bit word (low half = most recent tag), the slot
  // bit that no longer indexes joins the tag (htag + 1 <= 15 bits, so 0xFFFF stays "empty").  A hit
  // on the older way moves it to the front; a miss evicts the older way.  Lanes that race on one
  // set lose an insertion at worst (a later re-evaluation), never invent a tag
  if (TW && c.htag < 15) {
    uint32_t* h32 = reinterpret_cast<uint32_t*>(h) + (x >> (c.htag + 1));
    const uint32_t t = x & ((2u << c.htag) - 1u);
    const uint32_t w = *h32;
    const uint32_t lo = w & 0xffffu;
    if (lo == t) return false;
    *h32 = (lo << 16) | t;
    return (w >> 16) != t;
  }
#endif
  const uint32_t s = x >> c.htag;
  const uint16_t t = (uint16_t)(x & ((1u << c.htag) - 1u));
  if (h[s] == t) return false;
  h[s] = t;
  return true;
}

// gather row entries >= 0 of a -1 padded adjacency row into nb[] (compacted, order kept);
// if `h` is non-null, only ids newly inserted in the visited hash are kept.
__device__ __forceinline__ int gather_row(const int32_t* row, int cap, int32_t* nb, uint32_t* h, int hbits,
                                          int& fails, int& deg, int lane) {
  int m = 0;
  deg = 0;
  for (int t0 = 0; t0 < cap; t0 += 32) {
    const int j = t0 + lane;
    const int32_t u = j < cap ? __ldg(row + j) : -1;
    deg += __popc(__ballot_sync(kFull, u >= 0));
    bool keep = u >= 0;
    if (keep && h) keep = visit_new(h, hbits, u, fails);
    const uint32_t mask = __ballot_sync(kFull, keep);
    if (keep) nb[m + __popc(mask & ((1u << lane) - 1u))] = u;
    m += __popc(mask);
  }
  __syncwarp();
  return m;
}

// visited-bitmap test-and-set (atomicOr) with an L2 evict-last policy (AQR_VBM_HINT): every
// warp's bitmap is touched all over during a query (C4: ~20k of its 31k words), the bitmaps of
// the running queries together are about L2-sized, and the code rows streaming through L2 would
// otherwise evict them -- each test then became a DRAM round trip (C4: L2 hit rate 20%)
__device__ __forceinline__ uint64_t vbm_policy() {
  uint64_t pol = 0;
#if AQR_VBM_HINT
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
__device__ __forceinline__ uint32_t vbm_test_set(uint32_t* w, uint32_t bit, uint64_t pol) {
#if AQR_VBM_HINT
  uint32_t old;
  asm volatile("atom.global.or.L2::cache_hint.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(w), "r"(bit), "l"(pol) : "memory");
  return old;
#else
  return atomicOr(w, bit);
#endif
}

// AQR_VBM_LOAD: the bitmap word as L2 holds it (never L1: a line cached there could still hold
// the previous query's bits) / the bit set without waiting for the old value.  The bitmap is this
// warp's alone and a row holds no id twice, so the load decides the visit; a set a later load does
// not yet see could only cause a re-evaluation (R15), and __syncwarp orders them anyway
__device__ __forceinline__ uint32_t vbm_load(const uint32_t* w, uint64_t pol) {
  uint32_t v;
#if AQR_VBM_HINT
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(w), "l"(pol) : "memory");
#else
  v = __ldcg(w);
#endif
  return v;
}
__device__ __forceinline__ void vbm_set(uint32_t* w, uint32_t bit, uint64_t pol) {
#if AQR_VBM_HINT
  asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(w), "r"(bit), "l"(pol) : "memory");
#else
  atomicOr(w, bit);
#endif
}

// AQR_KW_HINT: position, after an insert of np sorted keys at insertion points slb[], of the first
// unexpanded W entry after new key 0, given that the old entries from slb[0] up to the old
// position kwpos (-1: none) are all expanded: min(new key 1 at slb[1] + 1, kwpos + #{j : slb[j] <=
// kwpos}); -2 when neither is inside the list after the insert (warp-uniform)
__device__ __forceinline__ int kw_hint(const int32_t* slb, int np, int kwpos, int size, int ef, int lane) {
  int h = np > 1 ? slb[1] + 1 : INT_MAX;
  if (kwpos >= 0) {
    int sft = 0;
    for (int j = lane; j < np; j += 32) sft += slb[j] <= kwpos;
#pragma unroll
    for (int off = 16; off; off >>= 1) sft += __shfl_xor_sync(kFull, sft, off);
    if (kwpos + sft < h) h = kwpos + sft;
  }
  const int nsize = size + np < ef ? size + np : ef;
  return h < nsize ? h : -2;
}

// rank sort of n 64-bit distinct keys: dst[rank(src[i])] = src[i]
__device__ __forceinline__ void rank_sort(const uint64_t* src, uint64_t* dst, int n, int lane) {
  for (int i = lane; i < n; i += 32) {
    const uint64_t k = src[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += src[j] < k;
    dst[r] = k;
  }
  __syncwarp();
}

// ------------------------------------------------------------------------------------
// fp32 distance of the query (smem, zero padded to d4) against one row, lanes own 4-wide
// chunks c = lane + 32 t; FMA per term; butterfly sum.  Stage 2 decodes the codes
// (x~ = xhat / scale + min, Alg2 l.11) and Stage 3 reads the fp32 row.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float a) {
#pragma unroll
  for (int off = 16; off; off >>= 1) a = __fadd_rn(a, __shfl_xor_sync(kFull, a, off));
  return a;
}

// a / s for a code a in [0, 255] from r = RN(1/s): one FMA correction of RN(a r)
__device__ __forceinline__ float div_code(float a, float s, float r) {
  const float q0 = __fmul_rn(a, r);
  return __fmaf_rn(__fmaf_rn(-q0, s, a), r, q0);
}

// every 128-byte line of [p, p + bytes) requested into L2 (no register result)
__device__ __forceinline__ void prefetch_l2_range(const void* p, uint32_t bytes) {
  const uint64_t a0 = reinterpret_cast<uint64_t>(p);
  for (uint64_t a = a0 & ~127ull; a < a0 + bytes; a += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}

// four rows at once (rows with id < 0 give 0), their loads in flight together.  Per row: lanes own
// 4-wide chunks c = lane + 32 t, one FMA per term in increasing c, then a butterfly sum.
// Stage 2 (EXACT = false) decodes the codes x~ = x^ / scale + min (IEEE division, Alg2 l.11);
// Stage 3 (EXACT = true) reads the fp32 row.
template <bool EXACT>
__device__ __forceinline__ void rows4(const IndexView& ix, const float* qf, const int32_t (&id)[4], int lane,
                                      float (&out)[4]) {
  const int n4 = ix.d4 >> 2;
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int c = lane; c < n4; c += 32) {
    const float4 qv = reinterpret_cast<const float4*>(qf)[c];
    float4 xv[4];
    if (EXACT) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        xv[r] = id[r] >= 0 ? __ldg(reinterpret_cast<const float4*>(ix.base + (int64_t)id[r] * ix.d4) + c)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        w[r] = id[r] >= 0 ? __ldg(reinterpret_cast<const uint32_t*>(ix.codes + (int64_t)id[r] * ix.d_pad) + c) : 0u;
      const float4 sv = __ldg(reinterpret_cast<const float4*>(ix.scale_j) + c);
      const float4 mv = __ldg(reinterpret_cast<const float4*>(ix.min_j) + c);
#pragma unroll
      if (AQR_FASTDIV && ix.fast_div) {
        // RN(a / s) as q0 = RN(a r), q = RN(q0 + RN(a - q0 s) r), r = RN(1/s) (Markstein's
        // correction; equality with the IEEE quotient verified for all 256 codes of every dimension
        // at upload, else the division below is used)
        const float4 rv = __ldg(reinterpret_cast<const float4*>(ix.rscale_j) + c);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          xv[r].x = __fadd_rn(div_code((float)(w[r] & 255u), sv.x, rv.x), mv.x);
          xv[r].y = __fadd_rn(div_code((float)((w[r] >> 8) & 255u), sv.y, rv.y), mv.y);
          xv[r].z = __fadd_rn(div_code((float)((w[r] >> 16) & 255u), sv.z, rv.z), mv.z);
          xv[r].w = __fadd_rn(div_code((float)(w[r] >> 24), sv.w, rv.w), mv.w);
        }
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          xv[r].x = __fadd_rn(__fdiv_rn((float)(w[r] & 255u), sv.x), mv.x);
          xv[r].y = __fadd_rn(__fdiv_rn((float)((w[r] >> 8) & 255u), sv.y), mv.y);
          xv[r].z = __fadd_rn(__fdiv_rn((float)((w[r] >> 16) & 255u), sv.z), mv.z);
          xv[r].w = __fadd_rn(__fdiv_rn((float)(w[r] >> 24), sv.w), mv.w);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (ix.metric == 0) {
        float e;
        e = __fsub_rn(qv.x, xv[r].x); acc[r] = __fmaf_rn(e, e, acc[r]);
        e = __fsub_rn(qv.y, xv[r].y); acc[r] = __fmaf_rn(e, e, acc[r]);
        e = __fsub_rn(qv.z, xv[r].z); acc[r] = __fmaf_rn(e, e, acc[r]);
        e = __fsub_rn(qv.w, xv[r].w); acc[r] = __fmaf_rn(e, e, acc[r]);
      } else {
        acc[r] = __fmaf_rn(qv.x, xv[r].x, acc[r]);
        acc[r] = __fmaf_rn(qv.y, xv[r].y, acc[r]);
        acc[r] = __fmaf_rn(qv.z, xv[r].z, acc[r]);
        acc[r] = __fmaf_rn(qv.w, xv[r].w, acc[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float a = warp_sum(acc[r]);
    out[r] = ix.metric == 0 ? a : __fsub_rn(1.0f, a);
  }
}

// adaptive re-rank depth (R27): the entries of A (sorted keys) with d^a <= (1 + tau_spread)
// d^a_k, at least k, at most `depth` -- a prefix of A, counted by ballots.  Out of line: inlined,
// it perturbed the register allocation of the whole search kernel (4.5% slower at C2 even when
// unused, measured)
__device__ __noinline__ int adaptive_depth(const uint64_t* akeys, int nc, int k, double tau_spread, int depth,
                                           int lane) {
  const int kk = k < nc ? k : nc;
  const double thr = __dmul_rn((double)fkey_inv((uint32_t)(akeys[kk - 1] >> 32)), __dadd_rn(1.0, tau_spread));
  int band = 0;
  for (int i0 = 0; i0 < nc; i0 += 32) {
    const int i = i0 + lane;
    const bool in = i < nc && (double)fkey_inv((uint32_t)(akeys[i] >> 32)) <= thr;
    band += __popc(__ballot_sync(kFull, in));
  }
  if (band < kk) band = kk;
  return band < depth ? band : depth;
}

// ------------------------------------------------------------------------------------
// Stages 2 / ET / 3 / assembly for one query (Alg2 l.8-24).  cid[0:nc] in smem holds C in
// (d^q, id) order; region holds >= 20*nc bytes of scratch after cid.
// ------------------------------------------------------------------------------------
// C comes either as ids (cid) or as the first nc W keys (wk, which may alias rkeys: entry i is
// read before it is overwritten).  akeys / rkeys: nc 64-bit keys each.
#if AQR_FINISH_NOINLINE
__device__ __noinline__
#else
__device__
#endif
void finish_query(const IndexView& ix, const SearchCfg& c, const float* qf, const int32_t* cid,
                             const uint64_t* wk, int nc, uint64_t* akeys, uint64_t* rkeys, int64_t qi,
                             int32_t* out_ids, float* out_dist, const aqr_debug& dbg, bool has_dbg, int lane,
                             int32_t* cnt) {
  // Stage 2: d^a for every entry of C (Alg2 l.10-12)
  if (AQR_PF_FINISH) {
    for (int i = lane; i < nc; i += 32) {
      const int32_t id = cid ? cid[i] : qkey_id(wk[i]);
      prefetch_l2_range(ix.codes + (int64_t)id * ix.d_pad, (uint32_t)ix.d_pad);
    }
  }
  for (int i0 = 0; i0 < nc; i0 += 4) {
    int32_t id[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) id[r] = i0 + r < nc ? (cid ? cid[i0 + r] : qkey_id(wk[i0 + r])) : -1;
#pragma unroll
    for (int r = 0; r < 4; ++r) AQR_ASSERT(id[r] < ix.n);
    float da[4];
    rows4<false>(ix, qf, id, lane, da);
    __syncwarp();  // wk may alias rkeys: these entries are read before they are overwritten
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (i0 + r < nc) rkeys[i0 + r] = akey(da[r], id[r]);
    }
  }
  __syncwarp();
  // A <- sort by (d^a, id) (Alg2 l.13)
  rank_sort(rkeys, akeys, nc, lane);
  // early termination (Alg2 l.15-16): fp64 test on the fp32 values (R11)
  const int k = c.k;
  int term = 0;
  if (c.early_term && nc > k) {
    const double ak = (double)fkey_inv((uint32_t)(akeys[k - 1] >> 32));
    const double ak1 = (double)fkey_inv((uint32_t)(akeys[k] >> 32));
    const double gap = __ddiv_rn(__dsub_rn(ak1, ak), __dadd_rn(ak, 1e-6));
    const double ratio = __ddiv_rn(ak1, __dadd_rn(ak, 1e-6));
    term = (gap > c.tau_gap) || (ratio > c.tau_ratio);
  }
  int depth = c.n_rerank < nc ? c.n_rerank : nc;
  if (AQR_ADAPTIVE && !isinf(c.tau_spread) && nc > 0) depth = adaptive_depth(akeys, nc, k, c.tau_spread, depth, lane);
  if (term && depth > k) depth = k;
  // Stage 3: exact distances for A[0:depth] (Alg2 l.19-22)
  if (AQR_PF_FINISH) {
    for (int i = lane; i < depth; i += 32)
      prefetch_l2_range(ix.base + (int64_t)(int32_t)(uint32_t)akeys[i] * ix.d4, 4u * (uint32_t)ix.d4);
  }
  for (int i0 = 0; i0 < depth; i0 += 4) {
    int32_t id[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) id[r] = i0 + r < depth ? (int32_t)(uint32_t)akeys[i0 + r] : -1;
    float de[4];
    rows4<true>(ix, qf, id, lane, de);
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (i0 + r < depth) {
          rkeys[i0 + r] = akey(de[r], id[r]);
          if (has_dbg && dbg.exact_d) dbg.exact_d[qi * c.n_coarse + i0 + r] = de[r];
        }
      }
    }
  }
  // assembly (Alg2 l.23-24): R = R_exact U (fill: as needed for k / union: the rest of A)
  int nr = depth;
  const int extra_end = c.assemble_mode == 0 ? (nc < k ? nc : k) : nc;
  for (int i = depth + lane; i < extra_end; i += 32) rkeys[i] = akeys[i];
  if (extra_end > nr) nr = extra_end;
  __syncwarp();
  if (has_dbg) {
    for (int i = lane; i < nc; i += 32) {
      if (dbg.asym_ids) dbg.asym_ids[qi * c.n_coarse + i] = (int32_t)(uint32_t)akeys[i];
      if (dbg.asym_d) dbg.asym_d[qi * c.n_coarse + i] = fkey_inv((uint32_t)(akeys[i] >> 32));
    }
  }
  __syncwarp();
  // sort R by (dist, id) into akeys (A no longer needed) and emit the top k
  rank_sort(rkeys, akeys, nr, lane);
  for (int t = lane; t < k; t += 32) {
    int32_t oid = -1;
    float od = INFINITY;
    if (t < nr) {
      oid = (int32_t)((int64_t)(int32_t)(uint32_t)akeys[t] + ix.id_base);
      od = fkey_inv((uint32_t)(akeys[t] >> 32));
    }
    out_ids[qi * k + t] = oid;
    out_dist[qi * k + t] = od;
  }
  if (lane == 0 && cnt) {
    cnt[6] = nc;
    cnt[7] = depth;
    cnt[8] = term;
    cnt[9] = nc;
  }
  __syncwarp();
}

__device__ __forceinline__ void load_query(const IndexView& ix, const float* q, int64_t ld_q, int64_t qi, float* qf,
                                           uint8_t* qc, int lane) {
  const float* qrow = q + qi * ld_q;
  for (int j = lane; j < ix.d4; j += 32) qf[j] = j < ix.d ? qrow[j] : 0.0f;
  __syncwarp();
  if (qc) {
    // Alg2 l.4: the same quantizer as the base vectors
    for (int j = lane; j < ix.d_pad; j += 32) {
      uint32_t code = 0;
      if (j < ix.d) {
        const float t = __fsub_rn(qf[j], __ldg(ix.min_j + j));
        const float u = __fmul_rn(t, __ldg(ix.scale_j + j));
        code = (uint32_t)roundf(fminf(fmaxf(u, 0.0f), 255.0f));
      }
      qc[j] = (uint8_t)code;
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------------------------------
// the fused search kernel
// ------------------------------------------------------------------------------------
// d^q for the rows of an INLINE block staged in shared memory (rows with id < 0 skipped)
template <int LPR, int CPL>
__device__ __forceinline__ void block_dists(const uint8_t* codes_s, int d_pad, const C32 (&qreg)[CPL], int qq,
                                            const int32_t* ids, int m, int32_t* out, int lane) {
  constexpr int G = 32 / LPR;
  constexpr int U = 4;
  const int g = lane / LPR, sub = lane % LPR;
  const int nch = d_pad >> 5;
  for (int r0 = 0; r0 < m; r0 += G * U) {
    C32 buf[U][CPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + g * U + u;
      const int id = r < m ? ids[r] : -1;
      const uint4* row = reinterpret_cast<const uint4*>(codes_s + (r < m ? r : 0) * d_pad);
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = sub + LPR * t;
        const bool ok = id >= 0 && c < nch;
        buf[u][t].a = ok ? row[2 * c] : make_uint4(0, 0, 0, 0);
        buf[u][t].b = ok ? row[2 * c + 1] : make_uint4(0, 0, 0, 0);
      }
    }
    int part[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      unsigned xx = 0, qx = 0;
#pragma unroll
      for (int t = 0; t < CPL; ++t) dp4a_c32(buf[u][t], qreg[t], xx, qx);
      part[u] = (int)xx - 2 * (int)qx;
    }
    reduce_rows<LPR, U>(part, sub);
    store_rows<LPR, U>(part, r0, g, sub, m, qq, out);
  }
}

// ------------------------------------------------------------------------------------
// the fused search kernel; INL selects the INLINE layer-0 layout (bulk-copied blocks,
// next block prefetched during the merge) or the GATHER layout (row + per-code gathers,
// shared-memory visited hash)
// ------------------------------------------------------------------------------------
template <int LPR, int CPL, bool INL, int CAP, bool FP, bool DBG>
__global__ void __launch_bounds__(32 * AQR_WARPS_PER_CTA, (LPR == 32 && AQR_WIDE_U > 0) ? 1 : AQR_MIN_CTAS) search_kernel(IndexView ix, SearchCfg c, Layout L, const float* __restrict__ q,
                                                     int64_t nq, int64_t ld_q, int32_t* __restrict__ out_ids,
                                                     float* __restrict__ out_dist, aqr_debug dbg, int dbg_flags,
                                                     int* __restrict__ counter) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  using H = Hot<LPR, CPL, CAP, nd_alias<LPR, INL, FP>()>;
  uint8_t* wb = smem + (threadIdx.x >> 5) * L.per_warp;
  uint8_t* qc = wb + L.o_qc;
  float* qf = reinterpret_cast<float*>(wb + L.o_qf);
  uint64_t* const Wbase = reinterpret_cast<uint64_t*>(wb + H::bytes);
  uint64_t* W = Wbase + AQR_W_SLACK;  // W[0] is Wbase[wstart]; set per query
  uint32_t* hash = reinterpret_cast<uint32_t*>(wb + L.o_h);
  int32_t* nb = reinterpret_cast<int32_t*>(wb + H::o_nb);
  int32_t* nd = reinterpret_cast<int32_t*>(wb + H::o_nd);
  uint64_t* cand = reinterpret_cast<uint64_t*>(wb + H::o_cand);
  uint64_t* cs = reinterpret_cast<uint64_t*>(wb + H::o_cs);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wb + H::o_bar);
  int32_t* clb = reinterpret_cast<int32_t*>(wb + H::o_lb);
  int32_t* scnt = reinterpret_cast<int32_t*>(wb + H::o_cnt);
  uint8_t* blkbuf = wb + L.o_h;
  uint8_t* stgbuf = wb + L.o_stg;  // the staged gather's rows (never overlaps the visited hash)
  uint32_t* vhash = c.hbits > 0 ? hash : nullptr;
  // visited_bits = -2: this warp slot's bitmap in global memory (exact; no shared memory)
  uint32_t* vbm = (!INL && c.vbm) ? c.vbm + ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * c.vbm_words
                                  : nullptr;
  const uint64_t vpol = vbm ? vbm_policy() : 0ull;
  const int sub = lane % LPR;
  const int nch = ix.d_pad >> 5;
  const int ef = c.ef;
  uint32_t phase = 0u;
  // wide rows: staged (TMA) gather, when the launcher chose it (c.staged)
  const bool STG = !INL && !FP && LPR == 32 && c.staged;
  // layer-0 scoring fused with the filter (list_filter) on the GATHER layout
  constexpr bool FUSE = !INL && !FP && AQR_FUSED_FILTER;
  uint32_t sph = 0u;                               // staged_dists parities (bit per buffer)
  if (INL || STG) {
    if (lane == 0) {
      mbar_init(bar, 1);
      if (STG) mbar_init(bar + 1, 1);
      fence_proxy_async();
    }
    __syncwarp();
  }

  // trace / counters requested (DBG = false: the timed instantiation, no debug code at all)
  const int has_dbg = DBG ? (dbg_flags & 1) : 0;
  for (;;) {
    int64_t qi = 0;
    if (lane == 0) qi = atomicAdd(counter, 1);
    qi = __shfl_sync(kFull, qi, 0);
    if (qi >= nq) break;
    if (DBG && (dbg_flags & 2) && lane == 0) dbg.t_ns[2 * qi] = globaltimer_ns();  // per-query latency
    // per-query counters live in shared memory and are only touched when a trace was requested,
    // so they cost no registers on the timed path
    int32_t* cnt = has_dbg ? scnt : nullptr;
    if (cnt && lane == 0) {
#pragma unroll
      for (int t = 0; t < AQR_NCOUNT; ++t) cnt[t] = 0;
    }
    int fails = 0;

    // 1. quantize the query
    load_query(ix, q, ld_q, qi, qf, FP ? nullptr : qc, lane);
    C32 qreg[CPL];
    int qq = 0;
    if (!FP) {
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int ch = sub + LPR * t;
        qreg[t].a = ch < nch ? reinterpret_cast<const uint4*>(qc)[2 * ch] : make_uint4(0, 0, 0, 0);
        qreg[t].b = ch < nch ? reinterpret_cast<const uint4*>(qc)[2 * ch + 1] : make_uint4(0, 0, 0, 0);
      }
      for (int j = lane; j < ix.d_pad; j += 32) qq += (int)qc[j] * (int)qc[j];
#pragma unroll
      for (int off = 16; off; off >>= 1) qq += __shfl_xor_sync(kFull, qq, off);
    }
    // distance keys of a list of node ids: d^q (the method) or the fp32 baseline's exact distance
    auto dists = [&](const int32_t* ids_, int m_, int32_t* out_) {
      if (FP) fp_dists<LPR>(ix, qf, ids_, m_, out_, lane);
      else if (LPR == 32 && STG) staged_dists<CPL>(ix, qreg, qq, ids_, m_, out_, lane, stgbuf, bar, sph);
      else list_dists<LPR, CPL>(ix, qreg, qq, ids_, m_, out_, lane);
    };

    // 2. greedy descent through the upper layers (R8)
    int32_t cur = ix.entry;
    if (lane == 0) nb[0] = cur;
    __syncwarp();
    dists(nb, 1, nd);
    __syncwarp();
    uint32_t dcur = (uint32_t)nd[0];
    if (cnt && lane == 0) cnt[5] += 1;
    for (int lv = ix.max_level; lv >= 1; --lv) {
      for (;;) {
        __syncwarp();
        const int32_t* row = ix.adj_up + (int64_t)(__ldg(ix.up_off + cur) + lv - 1) * ix.M;
        int deg;
        const int m = gather_row(row, ix.M, nb, nullptr, 0, fails, deg, lane);
        dists(nb, m, nd);
        __syncwarp();
        uint64_t best = qkey(dcur, cur);
        for (int r = lane; r < m; r += 32) {
          const uint64_t kk = qkey((uint32_t)nd[r], nb[r]);
          best = kk < best ? kk : best;
        }
        best = warp_min_u64(best);
        if (cnt && lane == 0) cnt[3] += 1;
        if (cnt && lane == 0) cnt[4] += deg;
        if (cnt && lane == 0) cnt[5] += m;
        if (qkey_id(best) == cur) break;
        cur = qkey_id(best);
        dcur = qkey_d(best);
      }
    }

    // 3. layer-0 beam (flag form)
    int wstart = AQR_W_SLACK;
    W = Wbase + wstart;
    if (INL) {
      if (lane == 0) {
        fence_proxy_async();
        bulk_load(blkbuf, ix.blk + (int64_t)cur * ix.blk_stride, (uint32_t)ix.blk_bytes, bar);
        W[0] = qkey(dcur, cur);
      }
    } else {
      if (vhash) {
        // empty: 0xFFFFFFFF (id slots) / 0xFFFF (16-bit tags)
        uint4* h4 = reinterpret_cast<uint4*>(hash);
        const int nh4 = ((c.htag >= 0 ? 2 : 4) << c.hbits) >> 4;
        for (int t = lane; t < nh4; t += 32) h4[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
      }
      if (vbm) {
        uint4* b4 = reinterpret_cast<uint4*>(vbm);
        for (int64_t t = lane; t < (c.vbm_words >> 2); t += 32) b4[t] = make_uint4(0, 0, 0, 0);
        __threadfence_block();
      }
      __syncwarp();
      if (lane == 0) {
        W[0] = qkey(dcur, cur);
        if (vhash) {
          if (c.htag >= 0) visit_new16<(AQR_HASH_2WAY > 0 && CAP > 56)>(reinterpret_cast<uint16_t*>(hash), c, cur);
          else visit_new(hash, c.hbits, cur, fails);
        }
        if (vbm) atomicOr(vbm + (cur >> 5), 1u << (cur & 31));
      }
    }
    __syncwarp();
    // GATHER: the layer-0 row of the node to expand next is held in registers (lane owns entries
    // lane + 32 t); it is loaded for the entry point here and, afterwards, prefetched for the next
    // expansion right after the filter so the load overlaps the merge
    constexpr int kRowRegs = (CAP + 31) / 32;  // cap0 = 2M <= CAP (56 or 160; ABI: M <= 80)
    int32_t arow[kRowRegs];
    int32_t arow2[kRowRegs];  // AQR_SPEC2: row of the guessed expansion after next
    if (!INL) {
#pragma unroll
      for (int t = 0; t < kRowRegs; ++t) {
        const int j = lane + 32 * t;
        arow[t] = -1;
        if (32 * t < ix.cap0 && j < ix.cap0) arow[t] = __ldg(ix.adj0 + (int64_t)cur * ix.ld0 + j);
      }
    }
    if (FUSE) {
      // list_filter reads whole passes of nb: entries no row fills stay -1
      for (int i = lane; i < H::NB; i += 32) nb[i] = -1;
      __syncwarp();
    }
    int size = 1, cursor = 0, nexp = 0;
    // AQR_KNOWN_NEXT: the position of the next expansion, known from the previous one (-1: scan
    // from the cursor, -2: W has no unexpanded entry left)
    int npos = -1;
    // AQR_KW_HINT: the first unexpanded W entry after the next expansion, when the insert told it
    // (-1: scan for it, -2: there is none).  Off in the one-warp kernel by default: in the
    // 128-byte-row kernels the extra live state cost C2 1.3% even when unused, and C4 (wide rows,
    // ef 2480) measured within its run-to-run noise (26.4-27.3 vs 26.4-27.1 ms); the cooperative
    // kernel keeps it (C3 ef 5888: 142.3 -> 136.1 ms)
    constexpr bool HINT = AQR_KW_HINT_SINGLE && AQR_KW_HINT > 0 && AQR_W_SLACK == 0 && !INL;
    int khint = -1, kwpos_l = -1;
    for (;;) {
      // smallest unexpanded entry of W
      int pos = -1, gpos = -1;
      if (AQR_KNOWN_NEXT && !AQR_SPEC2 && AQR_W_SLACK == 0 && npos != -1) {
        if (npos < 0) break;
        pos = npos;
      } else
      for (int bb = cursor; bb < size; bb += 32) {
        const int i = bb + lane;
        const bool un = i < size && !(W[i] & 1ull);
        const uint32_t mk = __ballot_sync(kFull, un);
        if (mk) {
          pos = bb + __ffs(mk) - 1;
          const uint32_t mk2 = mk & (mk - 1);
          if (mk2) gpos = bb + __ffs(mk2) - 1;
          break;
        }
      }
      if (pos < 0) break;
      // AQR_SPEC2: the next unexpanded entry is the following expansion unless this one inserts
      // a smaller key (~80% of expansions): load its row now, so that if it IS next its code
      // rows can be prefetched into L2 before this expansion's insert (side-effect free)
      int32_t spec = -1;
      if (!INL && AQR_SPEC2 && gpos >= 0) {
        spec = qkey_id(W[gpos]);
        const int64_t rb2 = (int64_t)spec * ix.ld0;
#pragma unroll
        for (int t = 0; t < kRowRegs; ++t) {
          const int j = lane + 32 * t;
          arow2[t] = -1;
          if (32 * t < ix.cap0 && j < ix.cap0) arow2[t] = __ldg(ix.adj0 + rb2 + j);
        }
      }
      AQR_ASSERT(pos >= 0 && pos < size && size <= ef);
      const uint64_t wk = W[pos];
      const int32_t cnode = qkey_id(wk);
      AQR_ASSERT(cnode >= 0 && cnode < ix.n && !(wk & 1ull));
      __syncwarp();
      if (lane == 0) {
        W[pos] = wk | 1ull;
        if (has_dbg && dbg.exp_ids && nexp < dbg.exp_cap) dbg.exp_ids[qi * dbg.exp_cap + nexp] = cnode;
      }
      ++nexp;
      uint64_t kw_e = ~0ull;
      int kwpos_e = -1;
      if (AQR_PF_ROW && !INL && !HINT) {
        // W does not change until the merge: find the next unexpanded entry now and pull its
        // adjacency row into L2 (no registers held); ~half of the expansions insert nothing, and
        // then this row's load would be fully exposed
        for (int bb = pos + 1; bb < size; bb += 32) {
          const int i = bb + lane;
          const bool un = i < size && !(W[i] & 1ull);
          const uint32_t mk = __ballot_sync(kFull, un);
          if (mk) {
            kwpos_e = bb + __ffs(mk) - 1;
            kw_e = W[kwpos_e];
            break;
          }
        }
        if (kwpos_e >= 0) {
          const uint64_t a0 = reinterpret_cast<uint64_t>(ix.adj0 + (int64_t)qkey_id(kw_e) * ix.ld0);
          const uint64_t a = (a0 & ~127ull) + 128ull * lane;
          if (a < a0 + 4ull * ix.cap0) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
        }
      }
      int m;
      const int32_t* ids;
      if (INL) {
        // the block of cnode was bulk-copied into blkbuf (prefetched during the last merge);
        // its ids are copied out so the buffer can take the next block before the merge
        mbar_wait(bar, phase);
        phase ^= 1u;
        m = ix.cap0;
        int deg = 0;
        for (int t0 = 0; t0 < m; t0 += 32) {
          const int32_t u = t0 + lane < m ? reinterpret_cast<const int32_t*>(blkbuf)[t0 + lane] : -1;
          if (t0 + lane < m) nb[t0 + lane] = u;
          deg += __popc(__ballot_sync(kFull, u >= 0));
        }
        ids = nb;
        if (cnt && lane == 0) cnt[1] += deg;
        if (cnt && lane == 0) cnt[2] += deg;
        block_dists<LPR, CPL>(blkbuf + ix.blk_ids, ix.d_pad, qreg, qq, reinterpret_cast<const int32_t*>(blkbuf), m,
                              nd, lane);
      } else {
        // neighbours (not yet visited, when the optional hash is on) from the prefetched row
        if (!AQR_PREFETCH_ROW) {
#pragma unroll
          for (int t = 0; t < kRowRegs; ++t) {
            const int j = lane + 32 * t;
            arow[t] = -1;
            if (32 * t < ix.cap0 && j < ix.cap0) arow[t] = __ldg(ix.adj0 + (int64_t)cnode * ix.ld0 + j);
          }
        }
        int deg = 0;
        m = 0;
        if (AQR_NOCOMPACT && !vhash && !vbm) {
          // the row as it is: -1 entries are skipped by the gather and the filter
          m = ix.cap0;
#pragma unroll
          for (int t = 0; t < kRowRegs; ++t) {
            AQR_ASSERT(arow[t] < ix.n && lane + 32 * t < H::NB);
            if (32 * t < ix.cap0) nb[lane + 32 * t] = arow[t];
          }
          if (has_dbg) {
#pragma unroll
            for (int t = 0; t < kRowRegs; ++t)
              if (32 * t < ix.cap0) deg += __popc(__ballot_sync(kFull, arow[t] >= 0));
          }
        } else if (vbm) {
          // visited bitmap: every test-and-set of the row in flight at once (one L2 round trip),
          // then the survivors (first visits) are compacted
          uint32_t old[kRowRegs];
#pragma unroll
          for (int t = 0; t < kRowRegs; ++t) {
            const int32_t u = arow[t];
            AQR_ASSERT(u < 0 || (u < ix.n && (int64_t)(u >> 5) < c.vbm_words));
            old[t] = (32 * t < ix.cap0 && u >= 0)
                         ? (AQR_VBM_LOAD ? vbm_load(vbm + (u >> 5), vpol) : vbm_test_set(vbm + (u >> 5), 1u << (u & 31), vpol))
                         : ~0u;
          }
#pragma unroll
          for (int t = 0; t < kRowRegs; ++t) {
            if (32 * t >= ix.cap0) break;  // uniform
            const int32_t u = arow[t];
            deg += __popc(__ballot_sync(kFull, u >= 0));
            const bool keep = u >= 0 && !(old[t] & (1u << (u & 31)));
            if (AQR_VBM_LOAD && keep) vbm_set(vbm + (u >> 5), 1u << (u & 31), vpol);
            const uint32_t mk = __ballot_sync(kFull, keep);
            AQR_ASSERT(!keep || m + __popc(mk & ((1u << lane) - 1u)) < H::NB);
            if (keep) nb[m + __popc(mk & ((1u << lane) - 1u))] = u;
            m += __popc(mk);
          }
        } else {
#pragma unroll
          for (int t = 0; t < kRowRegs; ++t) {
            if (32 * t >= ix.cap0) break;  // uniform
            const int32_t u = arow[t];
            deg += __popc(__ballot_sync(kFull, u >= 0));
            bool keep = u >= 0;
            if (keep && vhash)
              keep = c.htag >= 0 ? visit_new16<(AQR_HASH_2WAY > 0 && CAP > 56)>(reinterpret_cast<uint16_t*>(hash), c, u) : visit_new(hash, c.hbits, u, fails);
            const uint32_t mk = __ballot_sync(kFull, keep);
            AQR_ASSERT(!keep || m + __popc(mk & ((1u << lane) - 1u)) < H::NB);
            if (keep) nb[m + __popc(mk & ((1u << lane) - 1u))] = u;
            m += __popc(mk);
          }
        }
        if (FUSE && !(AQR_NOCOMPACT && !vhash && !vbm)) {
          // list_filter reads whole passes: -1 after the compacted ids
          for (int i = m + lane; i < (m + H::PASS - 1) / H::PASS * H::PASS; i += 32) nb[i] = -1;
        }
        __syncwarp();
        ids = nb;
        if (cnt && lane == 0) cnt[1] += deg;
        if (cnt && lane == 0) cnt[2] += (AQR_NOCOMPACT && !vhash && !vbm) ? deg : m;
        if (!(FUSE && !STG)) dists(nb, m, nd);
      }
      __syncwarp();
      // filter against max W (when full), then drop re-evaluations already in W (R15): the
      // survivors of the cheap key test are compacted first so the W binary search (which also
      // yields each candidate's insertion rank) runs once per survivor, not once per neighbour
      const uint64_t maxk = size >= ef ? (W[size - 1] & ~1ull) : ~0ull;
      int np0 = 0;
      if (FUSE && !STG) {
        np0 = list_filter<LPR, CPL>(ix, qreg, qq, ids, m, W, size, ef, cs, lane);
      } else
      for (int r0 = 0; r0 < m; r0 += 32) {
        const int r = r0 + lane;
        bool ok = false;
        uint64_t kk = 0;
        if (r < m) {
          const int32_t id = ids[r];
          kk = qkey((uint32_t)nd[r], id);
          ok = id >= 0 && kk < maxk;
        }
        const uint32_t mk = __ballot_sync(kFull, ok);
        if (ok) cs[np0 + __popc(mk & ((1u << lane) - 1u))] = kk;
        np0 += __popc(mk);
      }
      __syncwarp();
      int np = 0;
      uint64_t cmin = ~0ull;
      for (int j0 = 0; j0 < np0; j0 += 32) {
        const int j = j0 + lane;
        bool ok = false;
        uint64_t kk = 0;
        int lb = 0;
        if (j < np0) {
          kk = cs[j];
          lb = lower_bound_w(W, size, kk);
          ok = !(lb < size && (W[lb] & ~1ull) == kk);
        }
        const uint32_t mk = __ballot_sync(kFull, ok);
        if (ok) {
          const int jj = np + __popc(mk & ((1u << lane) - 1u));
          AQR_ASSERT(jj < CAP && lb >= 0 && lb <= size);
          cand[jj] = kk;
          clb[jj] = lb;
          cmin = kk < cmin ? kk : cmin;
        }
        np += __popc(mk);
      }
      if (cnt && lane == 0) cnt[11] += np0;
      if (cnt && lane == 0) cnt[12] += np;
      {
        // the next expansion is min(first unexpanded entry of W after pos, smallest candidate);
        // start loading its layer-0 data now so the load overlaps the merge (prefetch only,
        // never speculative: this node IS expanded next)
        if (!AQR_CMIN_GUARD || np > 0) cmin = warp_min_u64(cmin);  // np == 0: every lane holds ~0
        uint64_t kw = ~0ull;
        int kwpos = -1;
        if (HINT && khint != -1) {
          if (khint >= 0) {
            kwpos = khint;
            kw = W[khint];
          }
        } else if (AQR_PF_ROW && !INL && !HINT) {
          kwpos = kwpos_e;
          kw = kw_e;
        } else
        for (int bb = pos + 1; bb < size; bb += 32) {
          const int i = bb + lane;
          const bool un = i < size && !(W[i] & 1ull);
          const uint32_t mk = __ballot_sync(kFull, un);
          if (mk) {
            kwpos = bb + __ffs(mk) - 1;
            kw = W[kwpos];
            break;
          }
        }
        khint = -1;
        kwpos_l = kwpos;
        const uint64_t nxt = kw < cmin ? kw : cmin;
        // where the next expansion will sit after this one's merge: an old entry keeps its
        // position (every new key is larger than it), the smallest new key lands at its
        // insertion point slb[0]
        npos = nxt == ~0ull ? -2 : (kw < cmin ? kwpos : -3);
        __syncwarp();
        if (INL) {
          if (nxt != ~0ull && lane == 0) {
            fence_proxy_async();
            bulk_load(blkbuf, ix.blk + (int64_t)qkey_id(nxt) * ix.blk_stride, (uint32_t)ix.blk_bytes, bar);
          }
        } else if (AQR_PREFETCH_ROW && nxt != ~0ull) {
          if (spec >= 0 && qkey_id(nxt) == spec) {
            // guessed right: the row is here; pull its neighbours' code rows into L2 now
            const int lines = (ix.d_pad + 127) >> 7;
#pragma unroll
            for (int t = 0; t < kRowRegs; ++t) {
              arow[t] = arow2[t];
              if (32 * t < ix.cap0 && arow[t] >= 0) {
                const uint8_t* cr = ix.codes + (int64_t)arow[t] * ix.d_pad;
                for (int l = 0; l < lines; ++l) asm volatile("prefetch.global.L2 [%0];" ::"l"(cr + 128 * l));
              }
            }
          } else {
            const int64_t rb = (int64_t)qkey_id(nxt) * ix.ld0;
#pragma unroll
            for (int t = 0; t < kRowRegs; ++t) {
              const int j = lane + 32 * t;
              arow[t] = -1;
              if (32 * t < ix.cap0 && j < ix.cap0) arow[t] = ldg_first(ix.adj0 + rb + j);
            }
          }
        }
      }
      __syncwarp();
      if (np == 0) {
        cursor = pos + 1;
        continue;
      }
      // merge: sort the new keys (rank = #new keys below) into cs / slb; new key j lands at
      // slb[j] + j, and the old entries between consecutive insertion points, the segment
      // W[slb[j], slb[j+1]) (slb[np] = size), move right by j + 1 -- a constant per segment, so
      // each segment is a plain block move (top segment and top chunks first, in place; groups of
      // 4 chunks: one batch of loads, then one of stores).  Entries pushed to >= ef drop out.
      int32_t* slb = reinterpret_cast<int32_t*>(wb + H::o_slb);
      for (int i = lane; i < np; i += 32) {
        const uint64_t kk = cand[i];
        int r = 0;
#pragma unroll 4
        for (int j = 0; j < np; ++j) r += cand[j] < kk;
        AQR_ASSERT(r < np && np <= CAP);
        cs[r] = kk;
        slb[r] = clb[i];
      }
      __syncwarp();
      const int first_ins = slb[0];
      if (npos == -3) {
        npos = first_ins;
        // the new key 0 is expanded next; every old entry in [slb[0], kwpos) is already expanded
        // (pos was the smallest unexpanded, kwpos the first one after it), so the first unexpanded
        // entry after it is new key 1 (at slb[1] + 1) or the old kwpos entry, shifted by the insert
        if (HINT && ef >= AQR_KW_HINT) khint = kw_hint(slb, np, kwpos_l, size, ef, lane);
      }
      // move whichever side of the insertion points is shorter: the entries after the first
      // one right (tail), or those before the last one left into the free head slots (head)
      bool head = AQR_W_SLACK > 0 && slb[np - 1] < size - first_ins && np <= AQR_W_SLACK;
      if (head && wstart < np) {
        // re-centre: the whole list moves right so the head has AQR_W_SLACK free slots again
        const int sh = AQR_W_SLACK - wstart;
        for (int hi = size; hi > 0; hi -= 128) {
          const int lo = hi - 128 > 0 ? hi - 128 : 0;
          const int nchk = (hi - lo + 31) >> 5;
          uint64_t v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int p = lo + 32 * t + lane;
            if (t < nchk) v[t] = p < hi ? W[p] : 0ull;
          }
          __syncwarp();
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int p = lo + 32 * t + lane;
            if (t < nchk && p < hi) W[p + sh] = v[t];
          }
          __syncwarp();
        }
        W += sh;
        wstart += sh;
      }
      if (head) {
        // segment j = W[slb[j-1], slb[j]) (slb[-1] = 0) moves left by np - j, lowest first
        int seg_lo = 0;
        for (int j = 0; j < np; ++j) {
          const int sh = np - j;
          const int seg_hi2 = slb[j];
          for (int lo = seg_lo; lo < seg_hi2; lo += 128) {
            const int hi = lo + 128 < seg_hi2 ? lo + 128 : seg_hi2;
            uint64_t v[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int p = lo + 32 * t + lane;
              v[t] = p < hi ? W[p] : 0ull;
            }
            __syncwarp();
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int p = lo + 32 * t + lane;
              if (p < hi) W[p - sh] = v[t];
            }
            __syncwarp();
          }
          seg_lo = seg_hi2;
        }
        W -= np;
        wstart -= np;
      }
      int seg_hi = head ? 0 : size;
      bool flat = false;
#if AQR_FLAT_MERGE
      // many short segments (W still filling: ~40 new keys spread over a few hundred entries, ~30
      // instructions of loop overhead per segment): one top-down pass of 32-entry chunks instead,
      // each lane's shift = #{j : slb[j] <= p} by a binary search over the sorted slb
      if (!head && np * AQR_FLAT_MERGE > size - first_ins) {
        flat = true;
        for (int hi = size; hi > first_ins; hi -= 32) {
          const int p = hi - 32 + lane;
          uint64_t v = 0;
          int dst = -1;
          if (p >= first_ins) {
            v = W[p];
            int a = 0, b = np;
            while (a < b) {
              const int mid = (a + b) >> 1;
              if (slb[mid] <= p) a = mid + 1;
              else b = mid;
            }
            if (p + a < ef) dst = p + a;
          }
          __syncwarp();
          if (dst >= 0) W[dst] = v;
          __syncwarp();
        }
      }
#endif
      for (int j = (head || flat) ? -1 : np - 1; j >= 0; --j) {
        const int sh = j + 1;
        const int seg_lo = slb[j];
        int hi = seg_hi < ef - sh ? seg_hi : ef - sh;
#if AQR_SHORT_SEG
        if (hi - seg_lo <= 32) {
          // short segment (the common case): one chunk
          if (hi > seg_lo) {
            const int p = seg_lo + lane;
            const uint64_t v0 = p < hi ? W[p] : 0ull;
            __syncwarp();
            if (p < hi) W[p + sh] = v0;
            __syncwarp();
          }
          seg_hi = seg_lo;
          continue;
        }
#endif
#if AQR_MOVE32
        // 32 entries per step, top first: one load and one store per lane.  The store of a
        // step lands above its own loads (shift >= 1), never on entries still to be read, so
        // one __syncwarp (loads before stores) per step suffices
#if AQR_MOVE32 == 3
        // four unpredicated 32-entry chunks per step while the segment is long (C3 ef 4096: 265.9 ->
        // 253.5 ms; C2 ef 784: 9.76 -> 9.79, within noise.  Gated by a runtime ef test it cost C2 2.7%)
        for (; hi - 128 >= seg_lo; hi -= 128) {
          const uint64_t v3 = W[hi - 32 + lane], v2 = W[hi - 64 + lane], v1 = W[hi - 96 + lane],
                         v0 = W[hi - 128 + lane];
          __syncwarp();
          W[hi - 32 + lane + sh] = v3;
          W[hi - 64 + lane + sh] = v2;
          W[hi - 96 + lane + sh] = v1;
          W[hi - 128 + lane + sh] = v0;
        }
#endif
#if AQR_MOVE32 >= 2
        // two 32-entry chunks per step (64 entries: two loads in flight, one __syncwarp)
        for (; hi - 32 > seg_lo; hi -= 64) {
          const int p1 = hi - 32 + lane, p0 = hi - 64 + lane;
          const bool in0 = p0 >= seg_lo;
          const uint64_t v1 = W[p1];
          uint64_t v0 = 0;
          if (in0) v0 = W[p0];
          __syncwarp();
          AQR_ASSERT(p1 >= seg_lo && p1 + sh < ef);
          W[p1 + sh] = v1;
          if (in0) W[p0 + sh] = v0;
        }
        if (hi > seg_lo) {
          const int p = hi - 32 + lane;
          const bool in = p >= seg_lo;
          uint64_t v = 0;
          if (in) v = W[p];
          __syncwarp();
          if (in) W[p + sh] = v;
        }
#else
        for (; hi > seg_lo; hi -= 32) {
          const int p = hi - 32 + lane;
          const bool in = p >= seg_lo;
          uint64_t v = 0;
          if (in) v = W[p];
          __syncwarp();
          if (in) W[p + sh] = v;
        }
#endif
        __syncwarp();
        seg_hi = seg_lo;
        continue;
#endif
        for (; hi > seg_lo; hi -= 128) {
          const int lo = hi - 128 > seg_lo ? hi - 128 : seg_lo;
          uint64_t v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int p = lo + 32 * t + lane;
            v[t] = p < hi ? W[p] : 0ull;
          }
          __syncwarp();
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int p = lo + 32 * t + lane;
            if (p < hi) W[p + sh] = v[t];
          }
          __syncwarp();
        }
        seg_hi = seg_lo;
      }
      for (int j = lane; j < np; j += 32) {
        AQR_ASSERT(slb[j] >= 0 && slb[j] <= size);
        if (slb[j] + j < ef) W[slb[j] + j] = cs[j];
      }
      __syncwarp();
      size = size + np < ef ? size + np : ef;
      cursor = first_ins < pos + 1 ? first_ins : pos + 1;
    }
    if (cnt && lane == 0) cnt[0] = nexp;
    if (cnt && lane == 0) cnt[10] = fails;

    // debug: C with d^q
    const int nc = c.n_coarse < size ? c.n_coarse : size;
    __syncwarp();
    if (has_dbg) {
      for (int i = lane; i < c.n_coarse; i += 32) {
        const uint64_t wkk = i < nc ? W[i] : 0;
        if (dbg.coarse_ids) dbg.coarse_ids[qi * c.n_coarse + i] = i < nc ? qkey_id(wkk) : -1;
        if (dbg.coarse_dq)
          dbg.coarse_dq[qi * c.n_coarse + i] =
              i < nc ? (FP ? __float_as_int(fkey_inv(qkey_d(wkk))) : (int32_t)qkey_d(wkk)) : -1;
      }
    }
    if (FP) {
      // the baseline's result: the first k entries of W, distances exact already
      for (int t = lane; t < c.k; t += 32) {
        int32_t oid = -1;
        float od = INFINITY;
        if (t < size) {
          oid = (int32_t)((int64_t)qkey_id(W[t]) + ix.id_base);
          od = fkey_inv(qkey_d(W[t]));
        }
        out_ids[qi * c.k + t] = oid;
        out_dist[qi * c.k + t] = od;
      }
      if (has_dbg && lane == 0) {
        if (dbg.counters)
          for (int t = 0; t < AQR_NCOUNT; ++t) dbg.counters[qi * AQR_NCOUNT + t] = cnt[t];
        if (dbg.totals)
          for (int t = 0; t < AQR_NCOUNT; ++t)
            atomicAdd(reinterpret_cast<unsigned long long*>(dbg.totals + t), (unsigned long long)cnt[t]);
      }
      __syncwarp();
      continue;
    }
    if (L.q_alias) load_query(ix, q, ld_q, qi, qf, nullptr, lane);  // the beam reused its space
    // Stage 2/3 scratch lives in W: unsorted keys overwrite W[0:nc] in place, A goes to
    // W[nc:2nc] (ef >= 2 N_c, as with m_ef >= 2), else to a separate area
    uint64_t* akeys = ef >= 2 * nc ? W + nc : reinterpret_cast<uint64_t*>(wb + L.o_s23);
    uint64_t* rkeys = W;
    __syncwarp();
    // 4-7. Stage 2, early termination, Stage 3, assembly
    finish_query(ix, c, qf, nullptr, W, nc, akeys, rkeys, qi, out_ids, out_dist, dbg, has_dbg != 0, lane, cnt);
    if (has_dbg && lane == 0) {
      if (dbg.counters)
        for (int t = 0; t < AQR_NCOUNT; ++t) dbg.counters[qi * AQR_NCOUNT + t] = cnt[t];
      if (dbg.totals)
        for (int t = 0; t < AQR_NCOUNT; ++t) atomicAdd(reinterpret_cast<unsigned long long*>(dbg.totals + t),
                                                       (unsigned long long)cnt[t]);
    }
    __syncwarp();
    if (DBG && (dbg_flags & 2) && lane == 0) dbg.t_ns[2 * qi + 1] = globaltimer_ns();  // outputs written
  }
}

// ------------------------------------------------------------------------------------
// Cooperative search (aqr_search_params.warps_per_query = G > 1): one CTA of G warps per query,
// the same algorithm as search_kernel with the same results, visit order and counters (the
// parity tests run both).  For launches the one-warp kernel leaves latency-bound: a large ef
// (W alone limits an SM to a few queries: C3 ef 5888 -> 4 warps per SM) or few queries (C4:
// 1,000).  Per layer-0 expansion the G warps split
//   * the visited test of the row (one entry per thread) and its compaction (row order kept),
//   * the code gathers + dp4a scoring + max-W filter (list_filter) and the W dedupe: rows are
//     dealt round-robin, row r to warp r % G,
//   * the W insert: new keys ranked by all threads, the moved entries split into G contiguous
//     pieces (each warp saves its piece's bottom np entries -- the only ones the piece below can
//     overwrite -- then, after one barrier, block-moves the rest top-first in place and writes the
//     new keys whose insertion points lie in its piece);
// each warp finds the next expansion itself (all read the same W), so the next row is requested
// before the insert, as in search_kernel.  Warp 0 alone runs the greedy descent and Stages 2-3.
// ------------------------------------------------------------------------------------
#ifndef AQR_COOP_U
#define AQR_COOP_U 4  // rows per lane per scoring pass in the cooperative kernel
#endif

struct CoopMisc {
  long long qi;
  unsigned long long cmin[2];  // by expansion parity: one is filled while the other is reset
  int np[2], cur;
  unsigned dcur;
  int wcnt[16];
  int cnt[16];
  uint64_t bar[2];
};

struct CoopLayout {
  int o_w, o_nbw, nbw, o_sw, o_cand, o_clb, o_cs, o_slb, o_qc, o_qf, o_h, o_s23, bytes;
};

template <int LPR, int CPL>
__host__ __device__ constexpr int coop_pass() {
  return (32 / LPR) * AQR_COOP_U;
}

CoopLayout make_coop_layout(const IndexView& ix, const SearchCfg& c, int G, int cap, int pass) {
  CoopLayout L;
  int o = (int)((sizeof(CoopMisc) + 127) & ~(size_t)127);
  L.o_w = o; o += al16(8 * (c.ef + 1));
  const int per = (cap + G - 1) / G;
  L.nbw = (per + pass - 1) / pass * pass;  // one warp's id list, whole scoring passes
  if (L.nbw < 32) L.nbw = 32;
  L.o_nbw = o; o += al16(4 * G * L.nbw);
  L.o_sw = o; o += al16(8 * G * L.nbw);
  // cand doubles as the greedy descent's id list (rows of M <= 80 ids, padded to a pass)
  const int ncand = cap > 96 + pass ? cap : 96 + pass;
  L.o_cand = o; o += al16(8 * ncand);
  L.o_clb = o; o += al16(4 * cap);
  L.o_cs = o; o += al16(8 * ncand);
  L.o_slb = o; o += al16(4 * cap);
  L.o_qc = o; o += al16(ix.d_pad);
  L.o_qf = o; o += al16(4 * ix.d4);
  o = (o + 127) & ~127;
  L.o_h = o; o += c.hbits > 0 ? al16((c.htag >= 0 ? 2 : 4) << c.hbits) : 0;
  L.o_s23 = o; o += c.ef >= 2 * c.n_coarse ? 0 : al16(8 * c.n_coarse);
  L.bytes = (o + 127) & ~127;
  return L;
}

#ifndef AQR_COOP_MIN_CTAS
#define AQR_COOP_MIN_CTAS 5  // register budget of the cooperative kernel (4 warps: <= 102 registers)
#endif

template <int LPR, int CPL, int CAP, int G>
__global__ void __launch_bounds__(32 * G, AQR_COOP_MIN_CTAS) coop_kernel(IndexView ix, SearchCfg c, CoopLayout L,
                                                          const float* __restrict__ q, int64_t nq, int64_t ld_q,
                                                          int32_t* __restrict__ out_ids, float* __restrict__ out_dist,
                                                          aqr_debug dbg, int dbg_flags, int* __restrict__ counter) {
  constexpr int T = 32 * G;
  constexpr int RJ = (CAP + T - 1) / T;  // row entries per thread
  constexpr int PASS = coop_pass<LPR, CPL>();
  static_assert(RJ * G <= 16, "row slots");
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  CoopMisc* sm = reinterpret_cast<CoopMisc*>(smem);
  uint64_t* W = reinterpret_cast<uint64_t*>(smem + L.o_w);
  int32_t* nball = reinterpret_cast<int32_t*>(smem + L.o_nbw);
  int32_t* nbw = nball + w * L.nbw;  // this warp's id list
  uint64_t* sw = reinterpret_cast<uint64_t*>(smem + L.o_sw) + w * L.nbw;
  uint64_t* cand = reinterpret_cast<uint64_t*>(smem + L.o_cand);
  int32_t* clb = reinterpret_cast<int32_t*>(smem + L.o_clb);
  uint64_t* cs = reinterpret_cast<uint64_t*>(smem + L.o_cs);
  int32_t* slb = reinterpret_cast<int32_t*>(smem + L.o_slb);
  uint8_t* qc = smem + L.o_qc;
  float* qf = reinterpret_cast<float*>(smem + L.o_qf);
  uint32_t* vhash = c.hbits > 0 ? reinterpret_cast<uint32_t*>(smem + L.o_h) : nullptr;
  uint32_t* vbm = c.vbm ? c.vbm + (int64_t)blockIdx.x * c.vbm_words : nullptr;
  const uint64_t vpol = vbm ? vbm_policy() : 0ull;
  const bool nocomp = !vhash && !vbm;
  const int sub = lane % LPR;
  const int nch = ix.d_pad >> 5;
  const int ef = c.ef;
  const int has_dbg = dbg_flags & 1;
  int32_t* cnt = has_dbg ? sm->cnt : nullptr;
  // the id lists' slots past the row never get a row entry: -1 once (list_filter reads whole passes)
  for (int i = tid; i < G * L.nbw; i += T) nball[i] = -1;

  for (;;) {
    __syncthreads();
    if (tid == 0) sm->qi = atomicAdd(counter, 1);
    if (cnt && tid < 16) cnt[tid] = 0;
    __syncthreads();
    const int64_t qi = sm->qi;
    if (qi >= nq) break;
    if ((dbg_flags & 2) && tid == 0) dbg.t_ns[2 * qi] = globaltimer_ns();
    int fails = 0;
    // 1. the query (warp 0), the visited set's reset (all)
    if (w == 0) load_query(ix, q, ld_q, qi, qf, qc, lane);
    if (vhash) {
      uint4* h4 = reinterpret_cast<uint4*>(vhash);
      const int nh4 = ((c.htag >= 0 ? 2 : 4) << c.hbits) >> 4;
      for (int t = tid; t < nh4; t += T) h4[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    }
    if (vbm) {
      uint4* b4 = reinterpret_cast<uint4*>(vbm);
      for (int64_t t = tid; t < (c.vbm_words >> 2); t += T) b4[t] = make_uint4(0, 0, 0, 0);
      __threadfence_block();
    }
    __syncthreads();
    C32 qreg[CPL];
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int ch = sub + LPR * t;
      qreg[t].a = ch < nch ? reinterpret_cast<const uint4*>(qc)[2 * ch] : make_uint4(0, 0, 0, 0);
      qreg[t].b = ch < nch ? reinterpret_cast<const uint4*>(qc)[2 * ch + 1] : make_uint4(0, 0, 0, 0);
    }
    int qq = 0;
    for (int j = lane; j < ix.d_pad; j += 32) qq += (int)qc[j] * (int)qc[j];
#pragma unroll
    for (int off = 16; off; off >>= 1) qq += __shfl_xor_sync(kFull, qq, off);

    // 2. greedy descent through the upper layers (warp 0, R8)
    if (w == 0) {
      int32_t* gnb = reinterpret_cast<int32_t*>(cand);
      int32_t* gnd = reinterpret_cast<int32_t*>(cs);
      for (int i = lane; i < 2 * (L.o_clb - L.o_cand) / 8; i += 32) gnb[i] = -1;
      int32_t cur = ix.entry;
      if (lane == 0) gnb[0] = cur;
      __syncwarp();
      list_dists<LPR, CPL, AQR_COOP_U>(ix, qreg, qq, gnb, 1, gnd, lane);
      __syncwarp();
      uint32_t dcur = (uint32_t)gnd[0];
      if (cnt && lane == 0) cnt[5] += 1;
      for (int lv = ix.max_level; lv >= 1; --lv) {
        for (;;) {
          __syncwarp();
          const int32_t* row = ix.adj_up + (int64_t)(__ldg(ix.up_off + cur) + lv - 1) * ix.M;
          int deg;
          const int m = gather_row(row, ix.M, gnb, nullptr, 0, fails, deg, lane);
          list_dists<LPR, CPL, AQR_COOP_U>(ix, qreg, qq, gnb, m, gnd, lane);
          __syncwarp();
          uint64_t best = qkey(dcur, cur);
          for (int r = lane; r < m; r += 32) {
            const uint64_t kk = qkey((uint32_t)gnd[r], gnb[r]);
            best = kk < best ? kk : best;
          }
          best = warp_min_u64(best);
          if (cnt && lane == 0) {
            cnt[3] += 1;
            cnt[4] += deg;
            cnt[5] += m;
          }
          if (qkey_id(best) == cur) break;
          cur = qkey_id(best);
          dcur = qkey_d(best);
        }
      }
      if (lane == 0) {
        sm->cur = cur;
        sm->dcur = dcur;
        W[0] = qkey(dcur, cur);
        sm->np[0] = sm->np[1] = 0;
        sm->cmin[0] = sm->cmin[1] = ~0ull;
        if (vhash) {
          if (c.htag >= 0) visit_new16<(AQR_HASH_2WAY > 0 && CAP > 56)>(reinterpret_cast<uint16_t*>(vhash), c, cur);
          else visit_new(vhash, c.hbits, cur, fails);
        }
        if (vbm) atomicOr(vbm + (cur >> 5), 1u << (cur & 31));
      }
    }
    __syncthreads();

    // 3. layer-0 beam (flag form); row entry j of the node to expand is held by thread j % T
    int32_t myrow[RJ];
    {
      const int64_t rb = (int64_t)sm->cur * ix.ld0;
#pragma unroll
      for (int r = 0; r < RJ; ++r) {
        const int j = tid + T * r;
        myrow[r] = j < ix.cap0 ? __ldg(ix.adj0 + rb + j) : -1;
      }
    }
    int size = 1, cursor = 0, nexp = 0, npos = -1;
    int khint = -1, kwpos_l = -1;  // AQR_KW_HINT (as in search_kernel)
    for (;;) {
      // the smallest unexpanded entry of W (every warp: same W, same answer)
      int pos = -1;
      if (npos != -1) {
        if (npos < 0) break;
        pos = npos;
      } else {
        for (int bb = cursor; bb < size; bb += 32) {
          const int i = bb + lane;
          const uint32_t mk = __ballot_sync(kFull, i < size && !(W[i] & 1ull));
          if (mk) {
            pos = bb + __ffs(mk) - 1;
            break;
          }
        }
        if (pos < 0) break;
      }
      const uint64_t wk = W[pos];
      const int32_t cnode = qkey_id(wk);
      AQR_ASSERT(cnode >= 0 && cnode < ix.n && !(wk & 1ull));
      if (has_dbg && tid == 0 && dbg.exp_ids && nexp < dbg.exp_cap) dbg.exp_ids[qi * dbg.exp_cap + nexp] = cnode;
      const int par = nexp & 1;
      ++nexp;
      // the row: visited test + compaction (row order), dealt to the warps' lists (entry r -> warp r % G)
      int m;
      if (nocomp) {
        m = ix.cap0;
#pragma unroll
        for (int r = 0; r < RJ; ++r) {
          const int j = tid + T * r;
          AQR_ASSERT(j >= ix.cap0 || (j / G < L.nbw && myrow[r] < ix.n));
          if (j < ix.cap0) nball[(j % G) * L.nbw + j / G] = myrow[r];
          if (cnt) {
            const uint32_t mk = __ballot_sync(kFull, j < ix.cap0 && myrow[r] >= 0);
            if (lane == 0) {
              atomicAdd(cnt + 1, __popc(mk));
              atomicAdd(cnt + 2, __popc(mk));
            }
          }
        }
      } else {
        bool keep[RJ];
        uint32_t old[RJ];
        if (vbm) {
#pragma unroll
          for (int r = 0; r < RJ; ++r) {
            const int32_t u = myrow[r];
            old[r] = u >= 0 ? (AQR_VBM_LOAD ? vbm_load(vbm + (u >> 5), vpol) : vbm_test_set(vbm + (u >> 5), 1u << (u & 31), vpol))
                            : ~0u;
          }
        }
#pragma unroll
        for (int r = 0; r < RJ; ++r) {
          const int32_t u = myrow[r];
          if (vbm) {
            // (AQR_VBM_LOAD: the CTA's threads test distinct ids of one row, so the load decides)
            keep[r] = u >= 0 && !(old[r] & (1u << (u & 31)));
            if (AQR_VBM_LOAD && keep[r]) vbm_set(vbm + (u >> 5), 1u << (u & 31), vpol);
          }
          else keep[r] = u >= 0 && (c.htag >= 0 ? visit_new16<(AQR_HASH_2WAY > 0 && CAP > 56)>(reinterpret_cast<uint16_t*>(vhash), c, u)
                                                : visit_new(vhash, c.hbits, u, fails));
          const uint32_t mk = __ballot_sync(kFull, keep[r]);
          if (lane == 0) sm->wcnt[r * G + w] = __popc(mk);
          if (cnt) {
            const uint32_t md = __ballot_sync(kFull, u >= 0);
            if (lane == 0) atomicAdd(cnt + 1, __popc(md));
          }
        }
        __syncthreads();
        int tot = 0, base[RJ];
#pragma unroll
        for (int r = 0; r < RJ; ++r) base[r] = 0;
        for (int s = 0; s < RJ * G; ++s) {
          const int v = sm->wcnt[s];
#pragma unroll
          for (int r = 0; r < RJ; ++r)
            if (s < r * G + w) base[r] += v;
          tot += v;
        }
        m = tot;
#pragma unroll
        for (int r = 0; r < RJ; ++r) {
          const uint32_t mk = __ballot_sync(kFull, keep[r]);
          if (keep[r]) {
            const int rk = base[r] + __popc(mk & ((1u << lane) - 1u));
            AQR_ASSERT(rk < ix.cap0 && rk / G < L.nbw && myrow[r] < ix.n);
            nball[(rk % G) * L.nbw + rk / G] = myrow[r];
          }
        }
        if (cnt && tid == 0) atomicAdd(cnt + 2, m);
      }
      __syncthreads();
      // scoring + max-W filter + W dedupe of this warp's rows (W is read-only until the insert)
      const int mw = (m - w + G - 1) / G;
      if (!nocomp) {
        const int top = (mw + PASS - 1) / PASS * PASS;
        for (int i = mw + lane; i < top; i += 32) nbw[i] = -1;
        __syncwarp();
      }
      const int np0 = list_filter<LPR, CPL, AQR_COOP_U>(ix, qreg, qq, nbw, mw, W, size, ef, sw, lane);
      __syncwarp();
      uint64_t cminw = ~0ull;
      int npw = 0;
      for (int j0 = 0; j0 < np0; j0 += 32) {
        const int j = j0 + lane;
        bool ok = false;
        uint64_t kk = 0;
        int lb = 0;
        if (j < np0) {
          kk = sw[j];
          lb = lower_bound_w(W, size, kk);
          ok = !(lb < size && (W[lb] & ~1ull) == kk);
        }
        const uint32_t mk = __ballot_sync(kFull, ok);
        const int n = __popc(mk);
        int b0 = 0;
        if (lane == 0 && n) b0 = atomicAdd(&sm->np[par], n);
        b0 = __shfl_sync(kFull, b0, 0);
        if (ok) {
          const int jj = b0 + __popc(mk & ((1u << lane) - 1u));
          AQR_ASSERT(jj < CAP);
          cand[jj] = kk;
          clb[jj] = lb;
          cminw = kk < cminw ? kk : cminw;
        }
        npw += n;
      }
      cminw = warp_min_u64(cminw);
      if (lane == 0 && cminw != ~0ull) atomicMin(&sm->cmin[par], (unsigned long long)cminw);
      if (cnt && lane == 0) {
        atomicAdd(cnt + 11, np0);
        atomicAdd(cnt + 12, npw);
      }
      __syncthreads();
      // np / cmin of this expansion are complete; the other parity's pair is reset for the next
      // one (everyone read it before this expansion's first barrier).  W[pos]'s flag: nothing
      // reads it before the insert's barrier (the scans start at pos + 1, the dedupe masks it)
      if (tid == 0) {
        W[pos] = wk | 1ull;
        sm->np[par ^ 1] = 0;
        sm->cmin[par ^ 1] = ~0ull;
      }
      // the next expansion: min(first unexpanded entry after pos, smallest new key); its row is
      // requested now so the load overlaps the insert
      const int np = sm->np[par];
      {
        const uint64_t cmin = sm->cmin[par];
        uint64_t kw = ~0ull;
        int kwpos = -1;
        if (AQR_KW_HINT && khint != -1) {
          if (khint >= 0) {
            kwpos = khint;
            kw = W[khint];
          }
        } else
        for (int bb = pos + 1; bb < size; bb += 32) {
          const int i = bb + lane;
          const uint32_t mk = __ballot_sync(kFull, i < size && !(W[i] & 1ull));
          if (mk) {
            kwpos = bb + __ffs(mk) - 1;
            kw = W[kwpos];
            break;
          }
        }
        khint = -1;
        kwpos_l = kwpos;
        const uint64_t nxt = kw < cmin ? kw : cmin;
        npos = nxt == ~0ull ? -2 : (kw < cmin ? kwpos : -3);
        if (nxt != ~0ull) {
          const int64_t rb = (int64_t)qkey_id(nxt) * ix.ld0;
#pragma unroll
          for (int r = 0; r < RJ; ++r) {
            const int j = tid + T * r;
            myrow[r] = j < ix.cap0 ? ldg_first(ix.adj0 + rb + j) : -1;
          }
        }
      }
      if (np == 0) {
        // no insert: W is unchanged (but for the flag), so the next expansion may start at once
        cursor = pos + 1;
        continue;
      }
      // insert: rank the new keys (all threads), then move W top-down in rounds
      for (int i = tid; i < np; i += T) {
        const uint64_t kk = cand[i];
        int r = 0;
        for (int j = 0; j < np; ++j) r += cand[j] < kk;
        cs[r] = kk;
        slb[r] = clb[i];
      }
      __syncthreads();
      const int first_ins = slb[0];
      if (npos == -3) {
        npos = first_ins;
        if (AQR_KW_HINT && ef >= AQR_KW_HINT) khint = kw_hint(slb, np, kwpos_l, size, ef, lane);
      }
      {
        // the moved old entries [first_ins, size) split into G contiguous pieces, one per warp; each
        // warp first saves the bottom np entries of its piece (the stores of the piece below may land
        // there: an entry moves up by at most np), then, after one barrier, moves the rest top-first
        // in place by per-segment block moves (as search_kernel) and stores the saved entries
        constexpr int SV = (CAP + 31) / 32;
        const int per = (size - first_ins + G - 1) / G;
        const int a0 = first_ins + w * per;
        const int a1 = a0 + per < size ? a0 + per : size;
        const int nsv = a1 - a0 < np ? (a1 - a0 > 0 ? a1 - a0 : 0) : np;
        uint64_t svv[SV];
        int svd[SV];
#pragma unroll
        for (int t = 0; t < SV; ++t) {
          const int i = lane + 32 * t;
          svd[t] = -1;
          if (i < nsv) {
            const int p = a0 + i;
            svv[t] = W[p];
            int a = 0, b = np;  // shift = #{j : slb[j] <= p}
            while (a < b) {
              const int mid = (a + b) >> 1;
              if (slb[mid] <= p) a = mid + 1;
              else b = mid;
            }
            if (p + a < ef) svd[t] = p + a;
            AQR_ASSERT(p < size && a >= 1 && a <= np);
          }
        }
        __syncthreads();
        const int base = a0 + nsv;
        for (int j = np - 1; j >= 0; --j) {
          const int seg_top = j == np - 1 ? size : slb[j + 1];
          if (seg_top <= base) break;  // this segment and all below lie under the piece's moved part
          const int sh = j + 1;
          const int seg_lo = slb[j] > base ? slb[j] : base;
          int hi = seg_top < a1 ? seg_top : a1;
          if (hi > ef - sh) hi = ef - sh;
          AQR_ASSERT(seg_lo >= first_ins && (hi <= seg_lo || (hi <= size && hi + sh <= ef)));
          for (; hi - 128 >= seg_lo; hi -= 128) {
            const uint64_t v3 = W[hi - 32 + lane], v2 = W[hi - 64 + lane], v1 = W[hi - 96 + lane],
                           v0 = W[hi - 128 + lane];
            __syncwarp();
            W[hi - 32 + lane + sh] = v3;
            W[hi - 64 + lane + sh] = v2;
            W[hi - 96 + lane + sh] = v1;
            W[hi - 128 + lane + sh] = v0;
          }
          for (; hi > seg_lo; hi -= 32) {
            const int p = hi - 32 + lane;
            const bool in = p >= seg_lo;
            uint64_t v = 0;
            if (in) v = W[p];
            __syncwarp();
            if (in) W[p + sh] = v;
          }
          __syncwarp();
        }
#pragma unroll
        for (int t = 0; t < SV; ++t)
          if (svd[t] >= 0) W[svd[t]] = svv[t];
        // new key j goes to slb[j] + j, written by the warp whose piece holds its insertion point:
        // that slot is either in the warp's own (already moved) piece or among the next piece's
        // saved entries, so no other warp still has to read it
        __syncwarp();
        for (int j = lane; j < np; j += 32) {
          int own = per > 0 ? (slb[j] - first_ins) / per : 0;
          if (own > G - 1) own = G - 1;
          AQR_ASSERT(slb[j] >= first_ins && slb[j] <= size);
          if (own == w && slb[j] + j < ef) W[slb[j] + j] = cs[j];
        }
      }
      size = size + np < ef ? size + np : ef;
      cursor = first_ins < pos + 1 ? first_ins : pos + 1;
      __syncthreads();
    }
    if (cnt && tid == 0) {
      cnt[0] = nexp;
      cnt[10] = fails;
    }
    // 4-7. Stage 2, early termination, Stage 3, assembly (warp 0)
    const int nc = c.n_coarse < size ? c.n_coarse : size;
    if (w == 0) {
      if (has_dbg) {
        for (int i = lane; i < c.n_coarse; i += 32) {
          const uint64_t wkk = i < nc ? W[i] : 0;
          if (dbg.coarse_ids) dbg.coarse_ids[qi * c.n_coarse + i] = i < nc ? qkey_id(wkk) : -1;
          if (dbg.coarse_dq) dbg.coarse_dq[qi * c.n_coarse + i] = i < nc ? (int32_t)qkey_d(wkk) : -1;
        }
      }
      uint64_t* akeys = ef >= 2 * nc ? W + nc : reinterpret_cast<uint64_t*>(smem + L.o_s23);
      __syncwarp();
      finish_query(ix, c, qf, nullptr, W, nc, akeys, W, qi, out_ids, out_dist, dbg, has_dbg != 0, lane, cnt);
      if (has_dbg && lane == 0) {
        if (dbg.counters)
          for (int t = 0; t < AQR_NCOUNT; ++t) dbg.counters[qi * AQR_NCOUNT + t] = cnt[t];
        if (dbg.totals)
          for (int t = 0; t < AQR_NCOUNT; ++t)
            atomicAdd(reinterpret_cast<unsigned long long*>(dbg.totals + t), (unsigned long long)cnt[t]);
      }
      if ((dbg_flags & 2) && lane == 0) dbg.t_ns[2 * qi + 1] = globaltimer_ns();
    }
  }
}

// r_j = RN(1 / scale_j) and a check, for every code a in [0, 255], that div_code reproduces the
// IEEE quotient RN(a / scale_j) bit for bit (one thread per (j, a)); any mismatch sets *bad
__global__ void decode_recip_kernel(const float* __restrict__ scale, int32_t d4, float* __restrict__ rscale,
                                    int32_t* bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)d4 * 256) return;
  const int j = (int)(t >> 8);
  const float a = (float)(t & 255);
  const float s = scale[j];
  const float r = __frcp_rn(s);
  if ((t & 255) == 0) rscale[j] = r;
  if (__float_as_uint(div_code(a, s, r)) != __float_as_uint(__fdiv_rn(a, s))) atomicOr(bad, 1);
}

// |x^|^2 per node (exact int32: <= 255^2 * 2048 < 2^31), one thread per code row
__global__ void code_norms_kernel(IndexView ix, int32_t* __restrict__ out) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= ix.n) return;
  const uint4* row = reinterpret_cast<const uint4*>(ix.codes + v * ix.d_pad);
  unsigned acc = 0;
  for (int c = 0; c < (ix.d_pad >> 4); ++c) {
    const uint4 w = row[c];
    acc = __dp4a(w.x, w.x, acc);
    acc = __dp4a(w.y, w.y, acc);
    acc = __dp4a(w.z, w.z, acc);
    acc = __dp4a(w.w, w.w, acc);
  }
  out[v] = (int32_t)acc;
}

// INLINE layout builder: one warp per node copies its ids and its neighbours' code rows
__global__ void build_inline_kernel(IndexView ix, uint8_t* __restrict__ blk) {
  const int lane = threadIdx.x & 31;
  const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (v >= ix.n) return;
  uint8_t* out = blk + v * ix.blk_stride;
  const int32_t* row = ix.adj0 + v * ix.ld0;
  int32_t* oid = reinterpret_cast<int32_t*>(out);
  for (int t = lane; t < ix.blk_ids / 4; t += 32) oid[t] = t < ix.cap0 ? row[t] : -1;
  const int nch = ix.d_pad >> 4;
  uint4* oc = reinterpret_cast<uint4*>(out + ix.blk_ids);
  for (int e = lane; e < ix.cap0 * nch; e += 32) {
    const int r = e / nch, ch = e - r * nch;
    const int32_t u = row[r];
    oc[e] = u >= 0 ? reinterpret_cast<const uint4*>(ix.codes + (int64_t)u * ix.d_pad)[ch] : make_uint4(0, 0, 0, 0);
  }
}

// Stages 2 / ET / 3 / assembly alone, one warp per query
__global__ void __launch_bounds__(128) rerank_kernel(IndexView ix, SearchCfg c, const float* __restrict__ q,
                                                     int64_t nq, int64_t ld_q, const int32_t* __restrict__ cand,
                                                     int32_t n_cand, int32_t* __restrict__ out_ids,
                                                     float* __restrict__ out_dist, int per_warp, int o_reg) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (qi >= nq) return;
  uint8_t* wb = smem + (threadIdx.x >> 5) * per_warp;
  float* qf = reinterpret_cast<float*>(wb);
  int32_t* cid = reinterpret_cast<int32_t*>(wb + o_reg);
  load_query(ix, q, ld_q, qi, qf, nullptr, lane);
  // the list ends at the first -1
  int nc = n_cand;
  for (int b = 0; b < n_cand; b += 32) {
    const int i = b + lane;
    const bool end = i < n_cand && __ldg(cand + qi * n_cand + i) < 0;
    const uint32_t mk = __ballot_sync(kFull, end);
    if (mk) { nc = b + __ffs(mk) - 1; break; }
  }
  for (int i = lane; i < nc; i += 32) cid[i] = __ldg(cand + qi * n_cand + i);
  __syncwarp();
  uint64_t* akeys = reinterpret_cast<uint64_t*>(wb + o_reg + al16(4 * n_cand));
  uint64_t* rkeys = akeys + n_cand;
  aqr_debug none{};
  SearchCfg cc = c;
  cc.n_coarse = n_cand;
  finish_query(ix, cc, qf, cid, nullptr, nc, akeys, rkeys, qi, out_ids, out_dist, none, false, lane, nullptr);
}

template <int LPR, int CPL, int CAP, int G>
cudaError_t launch_coop(const IndexView& ix, const SearchCfg& cc, const float* q, int64_t nq, int64_t ld_q,
                        int32_t* out_ids, float* out_dist, const aqr_debug& d, int flags, int* counter, int nsm,
                        cudaStream_t s) {
  auto kern = coop_kernel<LPR, CPL, CAP, G>;
  const CoopLayout L = make_coop_layout(ix, cc, G, CAP, coop_pass<LPR, CPL>());
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * G, L.bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)nsm * per_sm;
  if (nq < grid) grid = nq;
  if (cc.vbm && grid > cc.vbm_slots) grid = cc.vbm_slots;  // one bitmap per CTA
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, 32 * G, L.bytes, s>>>(ix, cc, L, q, nq, ld_q, out_ids, out_dist, d, flags, counter);
  return cudaGetLastError();
}

// warps per query (include/aqr.h): one CTA of 4 warps per query where W alone limits an SM to <= 4
// one-warp queries (large ef: C3 at ef 5888, 165 -> 140 ms); measured no gain for C4's 1k queries
// at ef 2480 (26.6 vs 27.3 ms: two dependent memory round trips per expansion dominate either way)
// nor for C1's 100
int choose_wpq(int requested, int resident_warps_per_sm) {
  if (requested != 0) return requested;
  return resident_warps_per_sm <= 4 ? 4 : 1;
}

template <int LPR, int CPL, bool INL, int CAP, bool FP = false>
cudaError_t launch_t(const IndexView& ix, const SearchCfg& c, const float* q, int64_t nq, int64_t ld_q,
                     int32_t* out_ids, float* out_dist, const aqr_debug* dbg, int* counter, int wpb,
                     cudaStream_t s, int* plan = nullptr) {
  // plan != null: only report the warps per query this launch would use (no launch)
  if (plan) *plan = 1;
  // the flags decide before anything else: a launch without trace / counters / timestamps runs
  // the instantiation compiled without debug code (GATHER AQR traversal; the others keep one)
  aqr_debug d{};
  int flags = 0;
  if (dbg) {
    d = *dbg;
    if (d.exp_ids || d.coarse_ids || d.coarse_dq || d.asym_ids || d.asym_d || d.exact_d || d.counters || d.totals)
      flags |= 1;
    if (d.t_ns) flags |= 2;
  }
  auto kern = (!INL && !FP && flags == 0) ? search_kernel<LPR, CPL, INL, CAP, FP, INL || FP>
                                          : search_kernel<LPR, CPL, INL, CAP, FP, true>;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // resident warps for a configuration (per-warp shared memory at CTA size w)
  auto resident = [&](const Layout& Lx, int w, int* per_sm_out) -> cudaError_t {
    const size_t sm = (size_t)Lx.per_warp * w;
    cudaError_t er = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (er != cudaSuccess) return er;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm_out, kern, w * 32, sm);
  };
  SearchCfg cc = c;
  cc.staged = 0;
  hash_params(ix, cc);
  Layout L = make_layout(ix, cc, Hot<LPR, CPL, CAP, nd_alias<LPR, INL, FP>()>::bytes);
  if (L.per_warp > 12 * 1024) wpb = 1;  // large per-warp state: pack the SMs warp by warp
  int per_sm = 0;
  cudaError_t e = resident(L, wpb, &per_sm);
  if (e != cudaSuccess) return e;
  if (!INL && !FP && LPR == 32) {
    // wide code rows: stage them by TMA unless the stage costs concurrently running queries
    SearchCfg cs = cc;
    cs.staged = 1;
    const Layout Ls = make_layout(ix, cs, Hot<LPR, CPL, CAP, nd_alias<LPR, INL, FP>()>::bytes);
    const int ws = Ls.per_warp > 12 * 1024 ? 1 : wpb;
    int per_sm_s = 0;
    e = resident(Ls, ws, &per_sm_s);
    if (e != cudaSuccess) return e;
    const int64_t run0 = (int64_t)nsm * per_sm * wpb, run1 = (int64_t)nsm * per_sm_s * ws;
    const int64_t need = nq < run0 ? nq : run0;
    if (per_sm_s >= 1 && run1 >= need) {
      cc = cs;
      L = Ls;
      wpb = ws;
      per_sm = per_sm_s;
    }
  }
  e = resident(L, wpb, &per_sm);
  if (e != cudaSuccess) return e;
  if (plan && (INL || FP)) return cudaSuccess;
  if (!INL && !FP) {
    const int G = choose_wpq(c.wpq, per_sm * wpb);
    if (plan) {
      *plan = G;
      return cudaSuccess;
    }
    if (G == 4) {
      SearchCfg ck = cc;
      ck.staged = 0;
      return launch_coop<LPR, CPL, CAP, 4>(ix, ck, q, nq, ld_q, out_ids, out_dist, d, flags, counter, nsm, s);
    }
  }
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const size_t smem = (size_t)L.per_warp * wpb;
  int64_t want = (nq + wpb - 1) / wpb;
  int64_t grid = (int64_t)nsm * per_sm;
#if AQR_BALANCE
  // balance the rounds: with R = ceil(nq / resident warps) queries per warp, launch only
  // ceil(nq / R) warps, so the last round is (nearly) full instead of leaving most warps idle
  // while a few finish a partial round
  {
    const int64_t slots = grid * wpb;
    if (nq > slots) {
      const int64_t rounds = (nq + slots - 1) / slots;
      const int64_t warps = (nq + rounds - 1) / rounds;
      grid = (warps + wpb - 1) / wpb;
    }
  }
#endif
  if (want < grid) grid = want;
  if (cc.vbm && grid * wpb > cc.vbm_slots) grid = cc.vbm_slots / wpb;  // one bitmap per warp slot
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, wpb * 32, smem, s>>>(ix, cc, L, q, nq, ld_q, out_ids, out_dist, d, flags, counter);
  return cudaGetLastError();
}

// lanes per code row: the next power of two >= the row's 32-byte chunks, capped at 32 (each lane
// then loads CPL chunks of the row; d <= 2048 gives CPL <= 2); CAP: the adjacency-row class
struct Shape {
  int lpr, cpl, cap;
};
Shape shape_of(const IndexView& ix, bool fp = false) {
  const int nch = fp ? (ix.d4 >> 3) : (ix.d_pad >> 5);  // 32-byte chunks of a code / fp32 row
  if (fp) {
    int lpr = 1;
    while (lpr < nch) lpr <<= 1;
    if (lpr > 32) lpr = 32;
    return Shape{lpr, 1, ix.cap0 <= 56 ? 56 : 160};
  }
  int lpr = 1;
  while (lpr < nch) lpr <<= 1;
  if (lpr > 32) lpr = 32;
  return Shape{lpr, (nch + lpr - 1) / lpr, ix.cap0 <= 56 ? 56 : 160};
}

// F(lpr, cpl, cap) dispatch over the instantiated shapes
#define AQR_DISPATCH(SH, CALL)                                                      \
  switch ((SH).lpr * 1000 + (SH).cpl * 200 + (SH).cap) {                           \
    case 1256: CALL(1, 1, 56); case 1360: CALL(1, 1, 160);                        \
    case 2256: CALL(2, 1, 56); case 2360: CALL(2, 1, 160);                        \
    case 4256: CALL(4, 1, 56); case 4360: CALL(4, 1, 160);                        \
    case 8256: CALL(8, 1, 56); case 8360: CALL(8, 1, 160);                        \
    case 16256: CALL(16, 1, 56); case 16360: CALL(16, 1, 160);                    \
    case 32256: CALL(32, 1, 56); case 32360: CALL(32, 1, 160);                    \
    case 32456: CALL(32, 2, 56); case 32560: CALL(32, 2, 160);                    \
    default: break;                                                                \
  }

int hot_bytes(const IndexView& ix, bool fp) {
  const bool inl = ix.blk != nullptr;
#define AQR_HOT(L_, C_, K_)                                                   \
  return fp ? Hot<L_, C_, K_, nd_alias<L_, false, true>()>::bytes            \
            : inl ? Hot<L_, C_, K_, nd_alias<L_, true, false>()>::bytes      \
                  : Hot<L_, C_, K_, nd_alias<L_, false, false>()>::bytes
  AQR_DISPATCH(shape_of(ix, fp), AQR_HOT)
#undef AQR_HOT
  return -1;
}

}  // namespace

size_t search_smem_bytes(const IndexView& ix, const SearchCfg& c, int wpb) {
  const int hb = hot_bytes(ix, c.fp32 != 0);
  if (hb < 0) return ~(size_t)0;
  SearchCfg cc = c;
  hash_params(ix, cc);
  return (size_t)make_layout(ix, cc, hb).per_warp * wpb;
}

cudaError_t plan_search(const IndexView& ix, const SearchCfg& c, int64_t nq, int wpb, int* wpq) {
  *wpq = 1;
  if (c.fp32) return cudaSuccess;
  const bool inl = ix.blk != nullptr;
#define AQR_PLAN(L_, C_, K_)                                                                                  \
  return inl ? launch_t<L_, C_, true, K_>(ix, c, nullptr, nq, 0, nullptr, nullptr, nullptr, nullptr, wpb, 0, wpq) \
             : launch_t<L_, C_, false, K_>(ix, c, nullptr, nq, 0, nullptr, nullptr, nullptr, nullptr, wpb, 0, wpq)
  AQR_DISPATCH(shape_of(ix), AQR_PLAN)
#undef AQR_PLAN
  return cudaErrorInvalidValue;
}

cudaError_t launch_search(const IndexView& ix, const SearchCfg& c, const float* q, int64_t nq, int64_t ld_q,
                          int32_t* out_ids, float* out_dist, const aqr_debug* dbg, int* counter, int wpb,
                          cudaStream_t s) {
  if (c.fp32) {
    // the baseline runs the GATHER kernel (an INLINE index keeps its GATHER arrays)
#define AQR_LAUNCH_FP(L_, C_, K_) \
  return launch_t<L_, 1, false, K_, true>(ix, c, q, nq, ld_q, out_ids, out_dist, dbg, counter, wpb, s)
    const Shape sh = shape_of(ix, true);
    switch (sh.lpr * 1000 + sh.cap) {
      case 1056: AQR_LAUNCH_FP(1, 1, 56); case 1160: AQR_LAUNCH_FP(1, 1, 160);
      case 2056: AQR_LAUNCH_FP(2, 1, 56); case 2160: AQR_LAUNCH_FP(2, 1, 160);
      case 4056: AQR_LAUNCH_FP(4, 1, 56); case 4160: AQR_LAUNCH_FP(4, 1, 160);
      case 8056: AQR_LAUNCH_FP(8, 1, 56); case 8160: AQR_LAUNCH_FP(8, 1, 160);
      case 16056: AQR_LAUNCH_FP(16, 1, 56); case 16160: AQR_LAUNCH_FP(16, 1, 160);
      case 32056: AQR_LAUNCH_FP(32, 1, 56); case 32160: AQR_LAUNCH_FP(32, 1, 160);
      default: return cudaErrorInvalidValue;
    }
#undef AQR_LAUNCH_FP
  }
  const bool inl = ix.blk != nullptr;
#define AQR_LAUNCH(L_, C_, K_)                                                                            \
  return inl ? launch_t<L_, C_, true, K_>(ix, c, q, nq, ld_q, out_ids, out_dist, dbg, counter, wpb, s)    \
             : launch_t<L_, C_, false, K_>(ix, c, q, nq, ld_q, out_ids, out_dist, dbg, counter, wpb, s)
  AQR_DISPATCH(shape_of(ix), AQR_LAUNCH)
#undef AQR_LAUNCH
  return cudaErrorInvalidValue;
}

cudaError_t launch_decode_recip(const float* scale, int32_t d4, float* rscale, int32_t* bad, cudaStream_t s) {
  const int64_t n = (int64_t)d4 * 256;
  decode_recip_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(scale, d4, rscale, bad);
  return cudaGetLastError();
}

cudaError_t launch_code_norms(const IndexView& ix, int32_t* out, cudaStream_t s) {
  const int64_t grid = (ix.n + 255) / 256;
  code_norms_kernel<<<(unsigned)grid, 256, 0, s>>>(ix, out);
  return cudaGetLastError();
}

cudaError_t launch_build_inline(const IndexView& ix, uint8_t* blk, cudaStream_t s) {
  const int wpb = 8;
  const int64_t grid = (ix.n + wpb - 1) / wpb;
  build_inline_kernel<<<(unsigned)grid, wpb * 32, 0, s>>>(ix, blk);
  return cudaGetLastError();
}

cudaError_t launch_rerank(const IndexView& ix, const SearchCfg& c, const float* q, int64_t nq, int64_t ld_q,
                          const int32_t* cand, int32_t n_cand, int32_t* out_ids, float* out_dist,
                          cudaStream_t s) {
  const int wpb = 4;
  const int o_reg = al16(4 * ix.d4);
  const int per_warp = o_reg + al16(4 * n_cand) + al16(16 * n_cand + 16);
  const size_t smem = (size_t)per_warp * wpb;
  cudaError_t e = cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = (nq + wpb - 1) / wpb;
  rerank_kernel<<<(unsigned)grid, wpb * 32, smem, s>>>(ix, c, q, nq, ld_q, cand, n_cand, out_ids, out_dist,
                                                       per_warp, o_reg);
  return cudaGetLastError();
}

}  // namespace aqr
