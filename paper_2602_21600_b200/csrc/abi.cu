// abi.cu -- the C ABI of include/aqr.h: validation, ownership, launches.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

#include "aqr_internal.cuh"

struct aqr_index {
  aqr::IndexView v;
  int32_t layout = AQR_LAYOUT_GATHER;
  std::vector<void*> allocs;
  size_t bytes = 0;
};

namespace aqr {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

}  // namespace aqr

using aqr::set_error;

namespace {

#define AQR_CHECK_ARG(cond, msg)           \
  do {                                     \
    if (!(cond)) {                         \
      set_error(std::string("aqr: ") + msg); \
      return AQR_E_INVALID;                \
    }                                      \
  } while (0)

aqr_status cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string("aqr: CUDA error in ") + where + ": " + cudaGetErrorString(e));
  return (e == cudaErrorMemoryAllocation) ? AQR_E_OOM : AQR_E_CUDA;
}

#define AQR_CUDA(call, where)                   \
  do {                                          \
    cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

int32_t round_up(int32_t x, int32_t m) { return (x + m - 1) / m * m; }

}  // namespace

extern "C" {

const char* aqr_last_error(void) { return aqr::g_err.c_str(); }
#ifndef AQR_SRC_HASH
#define AQR_SRC_HASH "unknown"
#endif
// the build stamps the hash of the sources (paper_2602_21600_b200/build.py: src_hash)
const char* aqr_version(void) { return "aqr-b200 0.2 (sm_100a) src:" AQR_SRC_HASH; }

aqr_status aqr_encode(const float* x, int64_t n, int32_t d, int64_t ld_x, const aqr_train_cfg* train,
                      aqr_quant_params* qp, uint8_t* codes, aqr_stream_t stream) {
  aqr::g_err.clear();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  AQR_CHECK_ARG(x != nullptr && codes != nullptr && qp != nullptr, "encode: null pointer");
  AQR_CHECK_ARG(n >= 1 && d >= 1 && ld_x >= d, "encode: need n >= 1, d >= 1, ld_x >= d");
  AQR_CHECK_ARG(qp->d == d, "encode: qp->d != d");
  AQR_CHECK_ARG(qp->d_pad == round_up(d, 16), "encode: qp->d_pad must be round_up(d, 16)");
  AQR_CHECK_ARG(qp->min_j && qp->max_j && qp->scale_j, "encode: quantizer arrays must be allocated");
  if (train) {
    AQR_CHECK_ARG(train->sample_idx != nullptr, "encode: train->sample_idx is null");
    AQR_CHECK_ARG(train->k_density >= 1 && train->k_density <= 32, "encode: k_density must be in [1, 32]");
    AQR_CHECK_ARG(train->n_sample > train->k_density && train->n_sample <= n,
                  "encode: need k_density < n_sample <= n");
    AQR_CHECK_ARG(train->p_max >= 0.0 && train->p_max <= 50.0, "encode: p_max must be in [0, 50]");
    AQR_CHECK_ARG(train->eps > 0.0, "encode: eps must be > 0");
    AQR_CHECK_ARG(std::isnan(train->delta_override) ||
                      (train->delta_override >= 0.0 && train->delta_override <= 1.0),
                  "encode: delta_override must be NaN or in [0, 1]");
    double* meta = nullptr;
    double* rho = nullptr;
    void* tmp = nullptr;
    const bool need_rho = std::isnan(train->delta_override) || train->rho_out;
    // temporaries are released on every exit path (stream-ordered), including errors
    struct Tmp {
      double*& meta;
      double*& rho;
      void*& tmp;
      bool own_rho;
      cudaStream_t s;
      ~Tmp() {
        if (tmp) cudaFreeAsync(tmp, s);
        if (meta) cudaFreeAsync(meta, s);
        if (own_rho && rho) cudaFreeAsync(rho, s);
      }
    } guard{meta, rho, tmp, need_rho && !train->rho_out, s};
    AQR_CUDA(cudaMallocAsync((void**)&meta, 4 * sizeof(double), s), "encode: alloc");
    if (need_rho) {
      rho = train->rho_out;
      if (!rho) AQR_CUDA(cudaMallocAsync((void**)&rho, sizeof(double) * train->n_sample, s), "encode: alloc");
      AQR_CUDA(aqr::launch_density(x, ld_x, d, train->sample_idx, train->n_sample, train->k_density, train->eps,
                                   rho, s),
               "encode: density kernel");
    }
    AQR_CUDA(aqr::launch_delta(std::isnan(train->delta_override) ? rho : nullptr, train->n_sample, train->eps,
                               train->delta_override, train->p_max, meta, s),
             "encode: delta kernel");
    AQR_CUDA(cudaMallocAsync(&tmp, sizeof(float) * (size_t)n * d, s), "encode: alloc");
    AQR_CUDA(aqr::launch_train_columns(x, n, d, ld_x, meta, train->eps, qp->min_j, qp->max_j, qp->scale_j, tmp, s),
             "encode: percentile kernels");
    double hmeta[4] = {0, 0, 0, 0};
    AQR_CUDA(cudaMemcpyAsync(hmeta, meta, 3 * sizeof(double), cudaMemcpyDeviceToHost, s), "encode: copy");
    AQR_CUDA(cudaStreamSynchronize(s), "encode: sync");
    qp->delta = hmeta[0];
    qp->p_low = hmeta[1];
    qp->p_high = hmeta[2];
  }
  AQR_CUDA(aqr::launch_encode(x, n, d, ld_x, qp->min_j, qp->scale_j, codes, qp->d_pad, s), "encode: pack kernel");
  return AQR_OK;
}

aqr_status aqr_upload_index(const aqr_index_desc* desc, aqr_index** out, aqr_stream_t stream) {
  aqr::g_err.clear();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  AQR_CHECK_ARG(desc != nullptr && out != nullptr, "upload: null pointer");
  const aqr_index_desc& D = *desc;
  AQR_CHECK_ARG(D.n >= 1 && D.n < (int64_t(1) << 31), "upload: need 1 <= n < 2^31");
  AQR_CHECK_ARG(D.d >= 1, "upload: d >= 1");
  AQR_CHECK_ARG(D.d_pad == round_up(D.d, 16), "upload: d_pad must be round_up(d, 16)");
  AQR_CHECK_ARG(D.d_pad <= 2048, "upload: d > 2048 unsupported");
  AQR_CHECK_ARG(D.metric == AQR_L2 || D.metric == AQR_IP, "upload: bad metric");
  AQR_CHECK_ARG(D.codes && D.base && D.min_j && D.scale_j && D.adj0 && D.upper_off, "upload: null array");
  AQR_CHECK_ARG(D.ld_base >= D.d, "upload: ld_base < d");
  AQR_CHECK_ARG(D.M >= 1 && D.M <= 80, "upload: need 1 <= M <= 80 (layer-0 rows of <= 160 entries)");
  AQR_CHECK_ARG(D.max_level >= 0 && D.max_level <= 64, "upload: bad max_level");
  AQR_CHECK_ARG(D.entry_point >= 0 && D.entry_point < D.n, "upload: entry_point out of range");
  AQR_CHECK_ARG(D.upper_rows >= 0 && (D.upper_rows == 0 || D.adj_upper), "upload: adj_upper missing");
  AQR_CHECK_ARG(D.id_base >= 0 && D.id_base + D.n <= (int64_t(1) << 31), "upload: id_base + n must fit int32");
  AQR_CHECK_ARG(D.layout >= AQR_LAYOUT_AUTO && D.layout <= AQR_LAYOUT_INLINE, "upload: bad layout");
  const int64_t n = D.n;
  const int32_t cap0 = 2 * D.M, M = D.M;
  // host-side validation of the graph: ids in range, and no row lists a node twice or lists its
  // own node (a repeated id would be scored twice in one expansion and, having no visited set,
  // the kernel would insert both copies into W; the oracle's visited set would not)
  std::vector<int64_t> seen((size_t)n, -1);  // row stamp per node id
  for (int64_t v = 0; v < n; ++v) {
    for (int32_t t = 0; t < cap0; ++t) {
      const int32_t u = D.adj0[v * cap0 + t];
      AQR_CHECK_ARG(u >= -1 && u < n, "upload: adj0 id out of range");
      if (u < 0) continue;
      AQR_CHECK_ARG(u != v, "upload: adj0 row lists its own node (self-loop)");
      AQR_CHECK_ARG(seen[u] != v, "upload: adj0 row lists a neighbour twice");
      seen[u] = v;
    }
  }
  std::vector<int32_t> up_off((size_t)n);
  std::vector<int64_t> owner((size_t)(D.upper_rows > 0 ? D.upper_rows : 0), -1);
  for (int64_t v = 0; v < n; ++v) {
    AQR_CHECK_ARG(D.upper_off[v] >= -1 && D.upper_off[v] < D.upper_rows, "upload: upper_off out of range");
    up_off[v] = (int32_t)D.upper_off[v];
    if (D.upper_off[v] >= 0) owner[(size_t)D.upper_off[v]] = v;
  }
  // rows of a node are consecutive: a row without an owner of its own belongs to the one above
  for (int64_t r = 1; r < D.upper_rows; ++r)
    if (owner[(size_t)r] < 0) owner[(size_t)r] = owner[(size_t)r - 1];
  std::fill(seen.begin(), seen.end(), -1);
  for (int64_t r = 0; r < D.upper_rows; ++r) {
    for (int32_t t = 0; t < M; ++t) {
      const int32_t u = D.adj_upper[r * M + t];
      AQR_CHECK_ARG(u >= -1 && u < n, "upload: adj_upper id out of range");
      if (u < 0) continue;
      AQR_CHECK_ARG(u != owner[(size_t)r], "upload: adj_upper row lists its own node (self-loop)");
      AQR_CHECK_ARG(seen[u] != r, "upload: adj_upper row lists a neighbour twice");
      seen[u] = r;
    }
  }
  if (D.max_level > 0) {
    AQR_CHECK_ARG(D.upper_off[D.entry_point] >= 0 && D.upper_off[D.entry_point] + D.max_level <= D.upper_rows,
                  "upload: entry point must have level max_level");
  }
  aqr_index* ix = new aqr_index();
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes < 16 ? 16 : bytes) != cudaSuccess) return nullptr;
    ix->allocs.push_back(p);
    ix->bytes += bytes;
    return p;
  };
  auto fail = [&](aqr_status st) {
    aqr_index_free(ix);
    return st;
  };
  aqr::IndexView& V = ix->v;
  V.n = n;
  V.d = D.d;
  V.d_pad = round_up(D.d, 32);  // internal code stride: whole 32-byte chunks (one LDG.256 each)
  V.d4 = round_up(D.d, 8);  // fp32 row stride: whole 32-byte chunks (FP32 traversal loads 8 floats)
  V.metric = (int32_t)D.metric;
  V.id_base = D.id_base;
  V.M = M;
  V.cap0 = cap0;
  V.ld0 = round_up(cap0, 8);
  V.max_level = D.max_level;
  V.entry = D.entry_point;
  uint8_t* codes = (uint8_t*)alloc((size_t)n * V.d_pad);
  float* base = (float*)alloc(sizeof(float) * (size_t)n * V.d4);
  float* mn = (float*)alloc(sizeof(float) * V.d4);
  float* sc = (float*)alloc(sizeof(float) * V.d4);
  int32_t* a0 = (int32_t*)alloc(sizeof(int32_t) * (size_t)n * V.ld0);
  int32_t* au = (int32_t*)alloc(sizeof(int32_t) * (size_t)(D.upper_rows > 0 ? D.upper_rows * M : 1));
  int32_t* uo = (int32_t*)alloc(sizeof(int32_t) * (size_t)n);
  int32_t* xn = (int32_t*)alloc(sizeof(int32_t) * (size_t)n);
  if (!codes || !base || !mn || !sc || !a0 || !au || !uo || !xn) {
    set_error("aqr: upload: device allocation failed");
    return fail(AQR_E_OOM);
  }
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  if (V.d_pad != D.d_pad) chk(cudaMemsetAsync(codes, 0, (size_t)n * V.d_pad, s));
  chk(cudaMemcpy2DAsync(codes, V.d_pad, D.codes, D.d_pad, D.d_pad, n, cudaMemcpyDeviceToDevice, s));
  if (V.d4 != D.d) chk(cudaMemsetAsync(base, 0, sizeof(float) * (size_t)n * V.d4, s));
  chk(cudaMemcpy2DAsync(base, sizeof(float) * V.d4, D.base, sizeof(float) * D.ld_base, sizeof(float) * D.d, n,
                        cudaMemcpyDeviceToDevice, s));
  std::vector<float> ones(V.d4, 1.0f);
  chk(cudaMemsetAsync(mn, 0, sizeof(float) * V.d4, s));
  chk(cudaMemcpyAsync(sc, ones.data(), sizeof(float) * V.d4, cudaMemcpyHostToDevice, s));
  chk(cudaMemcpyAsync(mn, D.min_j, sizeof(float) * D.d, cudaMemcpyDeviceToDevice, s));
  chk(cudaMemcpyAsync(sc, D.scale_j, sizeof(float) * D.d, cudaMemcpyDeviceToDevice, s));
  chk(cudaMemsetAsync(a0, 0xff, sizeof(int32_t) * (size_t)n * V.ld0, s));
  chk(cudaMemcpy2DAsync(a0, sizeof(int32_t) * V.ld0, D.adj0, sizeof(int32_t) * cap0, sizeof(int32_t) * cap0, n,
                        cudaMemcpyHostToDevice, s));
  if (D.upper_rows > 0)
    chk(cudaMemcpyAsync(au, D.adj_upper, sizeof(int32_t) * (size_t)D.upper_rows * M, cudaMemcpyHostToDevice, s));
  chk(cudaMemcpyAsync(uo, up_off.data(), sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice, s));
  chk(cudaStreamSynchronize(s));
  if (e != cudaSuccess) {
    aqr_status st = cuda_fail(e, "upload");
    return fail(st);
  }
  V.codes = codes;
  V.xnorm = xn;
  V.base = base;
  V.min_j = mn;
  V.scale_j = sc;
  V.adj0 = a0;
  V.adj_up = au;
  V.up_off = uo;
  e = aqr::launch_code_norms(V, xn, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    aqr_status st = cuda_fail(e, "upload: code norms");
    return fail(st);
  }
  {
    // Stage 2 decode: reciprocal scales, and whether one FMA correction reproduces every quotient
    float* rs = (float*)alloc(sizeof(float) * V.d4);
    int32_t* bad = (int32_t*)alloc(sizeof(int32_t));
    if (!rs || !bad) {
      set_error("aqr: upload: device allocation failed");
      return fail(AQR_E_OOM);
    }
    int32_t bad_h = 1;
    e = cudaMemsetAsync(bad, 0, sizeof(int32_t), s);
    if (e == cudaSuccess) e = aqr::launch_decode_recip(sc, V.d4, rs, bad, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&bad_h, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      aqr_status st = cuda_fail(e, "upload: decode reciprocals");
      return fail(st);
    }
    V.rscale_j = rs;
    V.fast_div = bad_h == 0;
  }
  V.blk = nullptr;
  V.blk_ids = round_up(4 * cap0, 16);
  V.blk_bytes = V.blk_ids + cap0 * V.d_pad;
  V.blk_stride = (V.blk_bytes + 127) / 128 * 128;
  // layer-0 layout (include/aqr.h): AUTO = GATHER (measured faster on B200: the INLINE block
  // buffer costs occupancy and moves every neighbour row, profiles/r01)
  const size_t blk_total = (size_t)n * (size_t)V.blk_stride;
  const bool inl = D.layout == AQR_LAYOUT_INLINE;
  if (inl) {
    uint8_t* blk = (uint8_t*)alloc(blk_total);
    if (!blk) {
      set_error("aqr: upload: device allocation of the INLINE layout failed (use AQR_LAYOUT_GATHER)");
      return fail(AQR_E_OOM);
    }
    e = aqr::launch_build_inline(V, blk, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      aqr_status st = cuda_fail(e, "upload: inline layout");
      return fail(st);
    }
    V.blk = blk;
    ix->layout = AQR_LAYOUT_INLINE;
  }
  *out = ix;
  return AQR_OK;
}

void aqr_index_free(aqr_index* ix) {
  if (!ix) return;
  for (void* p : ix->allocs) cudaFree(p);
  delete ix;
}

size_t aqr_index_device_bytes(const aqr_index* ix) { return ix ? ix->bytes : 0; }
int32_t aqr_index_layout(const aqr_index* ix) { return ix ? ix->layout : 0; }

// 256 bytes (the persistent grid's query counter) + for visited_bits = -2 one n-bit visited bitmap
// per warp slot (at most one slot per query, and at most 64 resident warps per SM)
static int64_t vbm_words_of(const aqr_index* ix) { return ((ix->v.n + 127) / 128) * 4; }
static int64_t vbm_slots_of(int64_t nq) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cap = (int64_t)nsm * 64;
  const int64_t s = (nq + 3) / 4 * 4;
  return s < cap ? s : cap;
}

size_t aqr_search_workspace_size(const aqr_index* ix, int64_t nq, const aqr_search_params* p) {
  if (!ix || !p || p->visited_bits != -2 || nq <= 0) return 256;
  return 256 + (size_t)vbm_slots_of(nq) * (size_t)vbm_words_of(ix) * 4;
}

static aqr_status check_search_params(const aqr_search_params* p, bool need_ef) {
  AQR_CHECK_ARG(p != nullptr, "search: params null");
  AQR_CHECK_ARG(p->k >= 1 && p->k <= 1024, "search: need 1 <= k <= 1024");
  if (need_ef) {
    AQR_CHECK_ARG(p->n_coarse >= p->k, "search: need n_coarse >= k");
    AQR_CHECK_ARG(p->ef >= p->n_coarse, "search: need ef >= n_coarse");
    AQR_CHECK_ARG(p->ef <= 8192, "search: ef > 8192 unsupported");
    AQR_CHECK_ARG(p->n_rerank >= 0 && p->n_rerank <= p->n_coarse, "search: need 0 <= n_rerank <= n_coarse");
  } else {
    AQR_CHECK_ARG(p->n_rerank >= 0, "rerank: need n_rerank >= 0");
  }
  AQR_CHECK_ARG(p->tau_gap >= 0.0, "search: tau_gap must be >= 0");
  AQR_CHECK_ARG(p->tau_ratio >= 1.0, "search: tau_ratio must be >= 1");
  AQR_CHECK_ARG(p->tau_spread >= 0.0, "search: tau_spread must be >= 0 (INFINITY = static n_rerank)");
  AQR_CHECK_ARG(p->assemble_mode == 0 || p->assemble_mode == 1, "search: assemble_mode must be 0 or 1");
  AQR_CHECK_ARG(p->visited_bits == 0 || p->visited_bits == -1 || p->visited_bits == -2 ||
                    (p->visited_bits >= 6 && p->visited_bits <= 16),
                "search: visited_bits must be 0 (auto), -1 (no visited set), -2 (global bitmap) or in [6, 16]");
  AQR_CHECK_ARG(p->warps_per_block >= 0 && p->warps_per_block <= 8, "search: warps_per_block must be in [0, 8]");
  AQR_CHECK_ARG(p->traversal == AQR_TRAVERSAL_AQR || p->traversal == AQR_TRAVERSAL_FP32,
                "search: traversal must be AQR_TRAVERSAL_AQR (0) or AQR_TRAVERSAL_FP32 (1)");
  AQR_CHECK_ARG(p->warps_per_query == 0 || p->warps_per_query == 1 || p->warps_per_query == 4,
                "search: warps_per_query must be 0 (auto), 1 or 4");
  AQR_CHECK_ARG(p->warps_per_query <= 1 || p->traversal == AQR_TRAVERSAL_AQR,
                "search: warps_per_query 4 needs the AQR traversal");
  return AQR_OK;
}

static aqr::SearchCfg make_cfg(const aqr_search_params* p) {
  aqr::SearchCfg c;
  c.k = p->k;
  c.ef = p->ef;
  c.n_coarse = p->n_coarse;
  c.n_rerank = p->n_rerank;
  c.tau_gap = p->tau_gap;
  c.tau_ratio = p->tau_ratio;
  c.tau_spread = p->tau_spread;
  c.early_term = p->early_term;
  c.assemble_mode = p->assemble_mode;
  c.hbits = p->visited_bits > 0 ? p->visited_bits : 0;
  c.htag = -1;  // chosen per index by the launcher (hash_params)
  c.hmul = c.hmaskb = 0u;
  c.vbm = nullptr;  // visited_bits = -2: set by aqr_search from the workspace
  c.vbm_words = 0;
  c.vbm_slots = 0;
  c.fp32 = p->traversal == AQR_TRAVERSAL_FP32;
  c.staged = 0;  // chosen per launch by launch_search
  c.wpq = p->warps_per_query;
  return c;
}

aqr_status aqr_search(const aqr_index* ix, const float* q, int64_t nq, int64_t ld_q, const aqr_search_params* p,
                      int32_t* out_ids, float* out_dist, const aqr_debug* debug, void* ws, size_t ws_bytes,
                      aqr_stream_t stream) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(ix != nullptr, "search: index null");
  aqr_status st = check_search_params(p, true);
  if (st != AQR_OK) return st;
  AQR_CHECK_ARG(nq >= 0, "search: nq < 0");
  if (nq == 0) return AQR_OK;
  AQR_CHECK_ARG(q && out_ids && out_dist, "search: null pointer");
  AQR_CHECK_ARG(ld_q >= ix->v.d, "search: ld_q < d");
  AQR_CHECK_ARG(ws != nullptr && ws_bytes >= 256, "search: workspace too small");
  AQR_CHECK_ARG(!debug || !debug->exp_ids || debug->exp_cap >= 1, "search: debug exp_cap < 1");
  // the INLINE layout's beam reads each expansion's neighbours as one staged block and keeps no
  // visited set: a requested one would be ignored (and the bitmap would still shrink the grid)
  AQR_CHECK_ARG(!(ix->layout == AQR_LAYOUT_INLINE && p->traversal == AQR_TRAVERSAL_AQR &&
                  (p->visited_bits == -2 || p->visited_bits > 0)),
                "search: visited sets (visited_bits -2 or 6..16) need the GATHER layout");
  AQR_CHECK_ARG(!(ix->layout == AQR_LAYOUT_INLINE && p->traversal == AQR_TRAVERSAL_AQR && p->warps_per_query == 4),
                "search: warps_per_query 4 needs the GATHER layout");
  aqr::SearchCfg c = make_cfg(p);
#ifndef AQR_WARPS_PER_CTA
#define AQR_WARPS_PER_CTA 4
#endif
  int wpb = AQR_WARPS_PER_CTA;
  // one warp's state must fit a CTA (launch_search packs warps per CTA as shared memory allows)
  size_t smem = aqr::search_smem_bytes(ix->v, c, 1);
  if (smem > 227 * 1024) {
    set_error("aqr: search: per-warp shared memory exceeds 227 KB (reduce ef or visited_bits)");
    return AQR_E_UNSUPPORTED;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (p->visited_bits == -2) {
    c.vbm_words = vbm_words_of(ix);
    c.vbm_slots = (int64_t)((ws_bytes - 256) / 4 / (size_t)c.vbm_words);
    AQR_CHECK_ARG(c.vbm_slots >= 4, "search: workspace too small for the visited bitmaps (see aqr_search_workspace_size)");
    c.vbm = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + 256);
  }
  AQR_CUDA(cudaMemsetAsync(ws, 0, 256, s), "search: memset");
  AQR_CUDA(aqr::launch_search(ix->v, c, q, nq, ld_q, out_ids, out_dist, debug, static_cast<int*>(ws), wpb, s),
           "search: kernel launch");
  return AQR_OK;
}

aqr_status aqr_search_plan(const aqr_index* ix, int64_t nq, const aqr_search_params* p, int32_t* warps_per_query) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(ix != nullptr && warps_per_query != nullptr, "search_plan: null pointer");
  aqr_status st = check_search_params(p, true);
  if (st != AQR_OK) return st;
  AQR_CHECK_ARG(nq >= 0, "search_plan: nq < 0");
  aqr::SearchCfg c = make_cfg(p);
  int g = 1;
  AQR_CUDA(aqr::plan_search(ix->v, c, nq, AQR_WARPS_PER_CTA, &g), "search_plan: occupancy query");
  *warps_per_query = g;
  return AQR_OK;
}

aqr_status aqr_rerank(const aqr_index* ix, const float* q, int64_t nq, int64_t ld_q, const int32_t* cand_ids,
                      int32_t n_cand, const aqr_search_params* p, int32_t* out_ids, float* out_dist,
                      aqr_stream_t stream) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(ix != nullptr, "rerank: index null");
  aqr_status st = check_search_params(p, false);
  if (st != AQR_OK) return st;
  AQR_CHECK_ARG(nq >= 0 && n_cand >= 1 && n_cand <= 4096, "rerank: need nq >= 0, 1 <= n_cand <= 4096");
  if (nq == 0) return AQR_OK;
  AQR_CHECK_ARG(q && cand_ids && out_ids && out_dist, "rerank: null pointer");
  AQR_CHECK_ARG(ld_q >= ix->v.d, "rerank: ld_q < d");
  aqr::SearchCfg c = make_cfg(p);
  c.n_coarse = n_cand;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  AQR_CUDA(aqr::launch_rerank(ix->v, c, q, nq, ld_q, cand_ids, n_cand, out_ids, out_dist, s),
           "rerank: kernel launch");
  return AQR_OK;
}

aqr_status aqr_build_graph(const uint8_t* codes, int64_t n, int32_t d, int32_t d_pad, const int32_t* levels,
                           const int64_t* upper_off, int64_t upper_rows, int32_t M, int32_t efc, int32_t flags,
                           int32_t batch_div, int32_t* adj0, int32_t* adj_upper, int32_t* entry_max,
                           aqr_stream_t stream) {
  aqr::g_err.clear();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  AQR_CHECK_ARG(codes && levels && upper_off && adj0 && entry_max, "build: null pointer");
  AQR_CHECK_ARG(n >= 1 && n < (int64_t(1) << 31), "build: need 1 <= n < 2^31");
  AQR_CHECK_ARG(d >= 1 && d_pad == round_up(d, 16) && d_pad <= 2048, "build: need d_pad = round_up(d, 16) <= 2048");
  AQR_CHECK_ARG(M >= 2 && M <= 80, "build: need 2 <= M <= 80");
  AQR_CHECK_ARG(efc >= 1 && efc <= 1024, "build: need 1 <= efc <= 1024");
  AQR_CHECK_ARG(flags >= 0 && flags <= 3, "build: flags must be in [0, 3]");
  AQR_CHECK_ARG(batch_div >= 0, "build: batch_div must be >= 0");
  AQR_CHECK_ARG(upper_rows == 0 || adj_upper, "build: adj_upper missing");
  int64_t rows = 0;
  for (int64_t v = 0; v < n; ++v) {
    AQR_CHECK_ARG(levels[v] >= 0 && levels[v] <= 30, "build: levels must be in [0, 30]");
    AQR_CHECK_ARG(levels[v] == 0 ? upper_off[v] == -1 : upper_off[v] == rows,
                  "build: upper_off must list each node's rows consecutively, in node order (-1 for level 0)");
    rows += levels[v];
  }
  AQR_CHECK_ARG(rows == upper_rows && rows < (int64_t(1) << 31), "build: upper_rows must equal the sum of levels");
  const int32_t d32 = round_up(d, 32), cap0 = 2 * M;
  uint8_t* c32 = nullptr;
  int32_t *xn = nullptr, *lv = nullptr, *uo = nullptr, *a0 = nullptr, *au = nullptr;
  struct Free {  // device buffers are released on every exit path
    std::vector<void*> p;
    ~Free() {
      for (void* q : p) cudaFree(q);
    }
  } guard;
  auto alloc = [&](void** q, size_t bytes) -> cudaError_t {
    cudaError_t r = cudaMalloc(q, bytes < 16 ? 16 : bytes);
    if (r == cudaSuccess) guard.p.push_back(*q);
    return r;
  };
  AQR_CUDA(alloc((void**)&c32, (size_t)n * d32), "build: alloc");
  AQR_CUDA(alloc((void**)&xn, sizeof(int32_t) * (size_t)n), "build: alloc");
  AQR_CUDA(alloc((void**)&lv, sizeof(int32_t) * (size_t)n), "build: alloc");
  AQR_CUDA(alloc((void**)&uo, sizeof(int32_t) * (size_t)n), "build: alloc");
  AQR_CUDA(alloc((void**)&a0, sizeof(int32_t) * (size_t)n * cap0), "build: alloc");
  AQR_CUDA(alloc((void**)&au, sizeof(int32_t) * (size_t)(rows > 0 ? rows : 1) * M), "build: alloc");
  std::vector<int32_t> uo_h((size_t)n);
  for (int64_t v = 0; v < n; ++v) uo_h[(size_t)v] = (int32_t)upper_off[v];
  if (d32 != d_pad) AQR_CUDA(cudaMemsetAsync(c32, 0, (size_t)n * d32, s), "build: memset");
  AQR_CUDA(cudaMemcpy2DAsync(c32, d32, codes, d_pad, d_pad, n, cudaMemcpyDeviceToDevice, s), "build: codes");
  AQR_CUDA(cudaMemcpyAsync(lv, levels, sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice, s), "build: levels");
  AQR_CUDA(cudaMemcpyAsync(uo, uo_h.data(), sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice, s), "build: rows");
  AQR_CUDA(cudaMemsetAsync(a0, 0xff, sizeof(int32_t) * (size_t)n * cap0, s), "build: memset");
  AQR_CUDA(cudaMemsetAsync(au, 0xff, sizeof(int32_t) * (size_t)(rows > 0 ? rows : 1) * M, s), "build: memset");
  aqr::IndexView V{};
  V.n = n;
  V.codes = c32;
  V.d_pad = d32;
  AQR_CUDA(aqr::launch_code_norms(V, xn, s), "build: code norms");
  AQR_CUDA(aqr::build_graph_gpu(c32, xn, n, d32, lv, levels, uo, M, efc, flags, batch_div, a0, au, entry_max, s),
           "build: waves");
  AQR_CUDA(cudaMemcpyAsync(adj0, a0, sizeof(int32_t) * (size_t)n * cap0, cudaMemcpyDeviceToHost, s), "build: copy");
  if (rows > 0)
    AQR_CUDA(cudaMemcpyAsync(adj_upper, au, sizeof(int32_t) * (size_t)rows * M, cudaMemcpyDeviceToHost, s),
             "build: copy");
  AQR_CUDA(cudaStreamSynchronize(s), "build: sync");
  return AQR_OK;
}

aqr_status aqr_merge_topk(const float* dist, const int32_t* ids, int32_t n_lists, int64_t nq, int32_t k,
                          float* out_dist, int32_t* out_ids, aqr_stream_t stream) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(n_lists >= 1 && n_lists <= 32, "merge: need 1 <= n_lists <= 32");
  AQR_CHECK_ARG(k >= 1 && nq >= 0, "merge: need k >= 1, nq >= 0");
  if (nq == 0) return AQR_OK;
  AQR_CHECK_ARG(dist && ids && out_dist && out_ids, "merge: null pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  AQR_CUDA(aqr::launch_merge(dist, ids, n_lists, nq, k, out_dist, out_ids, s), "merge: kernel launch");
  return AQR_OK;
}

aqr_status aqr_peer_alloc(size_t bytes, void** dptr, uint8_t* handle) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(bytes > 0 && dptr != nullptr && handle != nullptr, "peer_alloc: need bytes > 0 and non-null outputs");
  static_assert(sizeof(cudaIpcMemHandle_t) == AQR_PEER_HANDLE_BYTES, "IPC handle size");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    set_error("aqr: peer_alloc: out of device memory");
    return AQR_E_OOM;
  }
  AQR_CUDA(e, "peer_alloc: cudaMalloc");
  e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(e, "peer_alloc: memset / cudaIpcGetMemHandle");
  }
  memcpy(handle, &h, sizeof(h));
  *dptr = p;
  return AQR_OK;
}

aqr_status aqr_peer_open(const uint8_t* handle, void** dptr) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(handle != nullptr && dptr != nullptr, "peer_open: null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  AQR_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "peer_open: cudaIpcOpenMemHandle");
  *dptr = p;
  return AQR_OK;
}

aqr_status aqr_peer_close(void* dptr) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(dptr != nullptr, "peer_close: null pointer");
  AQR_CUDA(cudaIpcCloseMemHandle(dptr), "peer_close: cudaIpcCloseMemHandle");
  return AQR_OK;
}

aqr_status aqr_peer_free(void* dptr) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(dptr != nullptr, "peer_free: null pointer");
  AQR_CUDA(cudaFree(dptr), "peer_free: cudaFree");
  return AQR_OK;
}

aqr_status aqr_peer_signal(uint64_t* const* flags, int32_t n_peers, int32_t slot, uint64_t value,
                           aqr_stream_t stream) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(flags != nullptr && n_peers >= 1 && n_peers <= AQR_MAX_PEERS, "peer_signal: need 1 <= n_peers <= 8");
  AQR_CHECK_ARG(slot >= 0, "peer_signal: slot < 0");
  for (int i = 0; i < n_peers; ++i) AQR_CHECK_ARG(flags[i] != nullptr, "peer_signal: null flag pointer");
  AQR_CUDA(aqr::launch_peer_signal(reinterpret_cast<unsigned long long* const*>(flags), n_peers, slot,
                                   (unsigned long long)value, reinterpret_cast<cudaStream_t>(stream)),
           "peer_signal: kernel launch");
  return AQR_OK;
}

aqr_status aqr_peer_wait(const uint64_t* flags, int32_t n, uint64_t value, uint64_t timeout_ns, int32_t* status,
                         aqr_stream_t stream) {
  aqr::g_err.clear();
  AQR_CHECK_ARG(flags != nullptr && n >= 1 && n <= 32, "peer_wait: need 1 <= n <= 32");
  AQR_CUDA(aqr::launch_peer_wait(reinterpret_cast<const unsigned long long*>(flags), n, (unsigned long long)value,
                                 (unsigned long long)timeout_ns, status, reinterpret_cast<cudaStream_t>(stream)),
           "peer_wait: kernel launch");
  return AQR_OK;
}

}  // extern "C"
