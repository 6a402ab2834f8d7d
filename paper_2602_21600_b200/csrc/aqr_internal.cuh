// aqr_internal.cuh -- shared declarations of the sm_100a implementation of include/aqr.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/aqr.h"

namespace aqr {

// Device-side view of an uploaded index (passed by value to kernels).
struct IndexView {
  int64_t n;
  int32_t d, d_pad, d4, metric;
  int64_t id_base;
  const uint8_t* codes;   // [n x d_pad]
  const int32_t* xnorm;   // [n] sum of squared codes |x^|^2 (d^q = |q^|^2 + |x^|^2 - 2 q^.x^)
  const float* base;      // [n x d4]   (d4 = round_up(d, 4), zero padded)
  const float* min_j;     // [d4]       (padding: 0)
  const float* scale_j;   // [d4]       (padding: 1)
  const float* rscale_j;  // [d4] RN(1 / scale_j): Stage 2 divides by one FMA correction step
  int32_t fast_div;       // 1: that step reproduces RN(x^ / scale_j) for every code (checked at upload)
  int32_t M, cap0, ld0;   // layer-0 rows: cap0 = 2M valid entries, stride ld0 (multiple of 8)
  const int32_t* adj0;    // [n x ld0]
  const int32_t* adj_up;  // [upper_rows x M]
  const int32_t* up_off;  // [n] (-1 for level-0 nodes)
  int32_t max_level, entry;
  // INLINE layout (nullptr for GATHER): per node a block of blk_stride bytes =
  // [cap0 int32 ids, padded to blk_ids bytes][cap0 code rows of d_pad bytes]
  const uint8_t* blk;
  int64_t blk_stride;
  int32_t blk_ids, blk_bytes;  // blk_bytes = blk_ids + cap0 * d_pad (bulk-copy size)
};

struct SearchCfg {
  int32_t k, ef, n_coarse, n_rerank;
  double tau_gap, tau_ratio;
  double tau_spread;      // adaptive re-rank depth (R27); +inf = static n_rerank
  int32_t early_term, assemble_mode;
  int32_t hbits;          // visited hash slots = 1 << hbits
  int32_t htag;           // set by the launcher: tag bits of the 16-bit-tag hash (-1: 32-bit id slots)
  uint32_t hmul, hmaskb;  // 16-bit-tag hash: odd multiplier and 2^B - 1 (2^B >= n)
  int32_t fp32;           // 1: FP32 baseline traversal (exact distances, no quantizer / re-rank)
  int32_t staged;         // set by the launcher: wide code rows gathered through a TMA stage
  int32_t wpq;            // warps per query: 0 auto, 1 one warp, 4 a cooperative CTA (coop_kernel)
  uint32_t* vbm;          // visited_bits = -2: per-warp-slot visited bitmaps (workspace), else null
  int64_t vbm_words;      // 32-bit words per bitmap (multiple of 4)
  int64_t vbm_slots;      // bitmaps available (bounds the persistent grid's warps)
};

void set_error(const std::string& msg);

// launchers (defined in encode.cu / search.cu / merge.cu); return cudaError_t of the launch
cudaError_t launch_density(const float* x, int64_t ld_x, int32_t d, const int32_t* sample, int32_t ns,
                           int32_t k, double eps, double* rho, cudaStream_t s);
cudaError_t launch_delta(const double* rho, int32_t ns, double eps, double delta_override, double p_max,
                         double* meta /*device [3]*/, cudaStream_t s);
cudaError_t launch_train_columns(const float* x, int64_t n, int32_t d, int64_t ld_x, const double* meta,
                                 double eps, float* min_j, float* max_j, float* scale_j, void* tmp,
                                 cudaStream_t s);
cudaError_t launch_encode(const float* x, int64_t n, int32_t d, int64_t ld_x, const float* min_j,
                          const float* scale_j, uint8_t* codes, int32_t d_pad, cudaStream_t s);
cudaError_t launch_decode_recip(const float* scale, int32_t d4, float* rscale, int32_t* bad, cudaStream_t s);
cudaError_t launch_search(const IndexView& ix, const SearchCfg& c, const float* q, int64_t nq, int64_t ld_q,
                          int32_t* out_ids, float* out_dist, const aqr_debug* dbg, int* counter,
                          int warps_per_block, cudaStream_t s);
cudaError_t launch_rerank(const IndexView& ix, const SearchCfg& c, const float* q, int64_t nq, int64_t ld_q,
                          const int32_t* cand, int32_t n_cand, int32_t* out_ids, float* out_dist,
                          cudaStream_t s);
cudaError_t launch_merge(const float* dist, const int32_t* ids, int32_t n_lists, int64_t nq, int32_t k,
                         float* out_dist, int32_t* out_ids, cudaStream_t s);
size_t search_smem_bytes(const IndexView& ix, const SearchCfg& c, int warps_per_block);
cudaError_t plan_search(const IndexView& ix, const SearchCfg& c, int64_t nq, int warps_per_block, int* wpq);
cudaError_t launch_peer_signal(unsigned long long* const* flags, int n_peers, int slot, unsigned long long value,
                               cudaStream_t s);
cudaError_t launch_peer_wait(const unsigned long long* flags, int n, unsigned long long value,
                             unsigned long long timeout_ns, int32_t* status, cudaStream_t s);
cudaError_t launch_build_inline(const IndexView& ix, uint8_t* blk, cudaStream_t s);
cudaError_t launch_code_norms(const IndexView& ix, int32_t* out, cudaStream_t s);
// GPU index build (build.cu): codes [n x d_pad32] (d_pad32 a multiple of 32, zero padded), their
// |x^|^2, levels on device and host, upper_off on device (int32); fills adj0_d [n x 2M] and adj_up_d
// (both pre-set to -1) and entry_max (host) = {entry point, top level}
cudaError_t build_graph_gpu(const uint8_t* codes, const int32_t* xnorm, int64_t n, int32_t d_pad32,
                            const int32_t* levels_d, const int32_t* levels_h, const int32_t* up_off_d, int32_t M,
                            int32_t efc, int32_t flags, int32_t batch_div, int32_t* adj0_d, int32_t* adj_up_d,
                            int32_t* entry_max, cudaStream_t s);
size_t build_smem_bytes(int32_t efc);

}  // namespace aqr
