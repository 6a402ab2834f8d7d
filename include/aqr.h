/*
 * aqr.h -- C ABI of the B200-native AQR-HNSW hot path (arXiv 2602.21600).
 *
 * The boundary of the batched k-NN query search of AQR-HNSW: density-aware uint8
 * quantization (Alg1 Stages 1-2), the HNSW index upload (Alg1 Stage 3
 * output), the fused search (Alg2) and the cross-shard merge
 * (BASELINE.json configs[4]).  Citations: P:n = PAPER.md line n; "Alg2 l.k" = Algorithm 2's
 * own line k; R<n> = a reading recorded in DESIGN.md "Readings of the paper".
 *
 * Conventions for every entry point
 *  - Pointers documented "device" must be CUDA device pointers (cudaMalloc / torch CUDA
 *    tensors) on the current device; "host" pointers are ordinary CPU memory.  All arrays are
 *    dense row-major.  The caller owns every array it passes; the library never frees them.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are asynchronous on
 *    that stream unless documented otherwise.
 *  - No exception crosses the ABI.  Every call returns an aqr_status; on failure
 *    aqr_last_error() returns a thread-local message describing the first failure.
 *    Argument errors are detected on the host before anything is launched (AQR_E_INVALID).
 *    Kernel faults surface as AQR_E_CUDA at the call that observes them.
 *  - Ties are broken by (value, id) ascending everywhere.
 */
#ifndef AQR_H_
#define AQR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *aqr_stream_t; /* == cudaStream_t */

typedef enum {
  AQR_OK = 0,
  AQR_E_INVALID = 1,     /* bad argument (host-side validation) */
  AQR_E_CUDA = 2,        /* CUDA runtime / kernel error */
  AQR_E_OOM = 3,         /* device allocation failed */
  AQR_E_UNSUPPORTED = 4, /* configuration outside what the kernels support */
  AQR_E_STATE = 5        /* object used in the wrong state */
} aqr_status;

typedef enum { AQR_L2 = 0, AQR_IP = 1 } aqr_metric;

/* ------------------------------------------------------------------------------------ */
/* aqr_encode -- density-aware u8 quantization (Alg1 l.5-11)          */
/* ------------------------------------------------------------------------------------ */

/* Quantizer parameters.  min_j / max_j / scale_j are DEVICE arrays of length d allocated by
 * the caller.  When the quantizer is trained by aqr_encode they are written; otherwise they
 * are read.  delta / p_low / p_high are written on the host when training. */
typedef struct {
  int32_t d;        /* dimensionality */
  int32_t d_pad;    /* code row stride in bytes: the smallest multiple of 16 that is >= d */
  float *min_j;     /* device [d]: P_l percentile of dimension j */
  float *max_j;     /* device [d]: P_h percentile of dimension j */
  float *scale_j;   /* device [d]: 255 / (max_j - min_j + eps) (Alg1 l.11); 1 if degenerate */
  double delta;     /* heterogeneity (Alg1 l.6) */
  double p_low;     /* P_l = delta * P_max (Alg1 l.8, percent scale R3) */
  double p_high;    /* P_h = 100 - delta * P_max */
} aqr_quant_params;

/* Training configuration.  The density sample (when n > 10,000, n_s = min(5000, n)
 * points, else all points) is drawn by the caller from its seed and passed in sorted. */
typedef struct {
  const int32_t *sample_idx; /* device [n_sample], sorted ascending, distinct, in [0, n) */
  int32_t n_sample;          /* > k_density */
  int32_t k_density;         /* kNN size for the density ("typically k = 10") */
  double p_max;              /* maximum percentile width P_max (R4; default 5) */
  double eps;                /* epsilon (1e-6) */
  double delta_override;     /* NaN => compute delta from the sample, else use this value */
  double *rho_out;           /* optional device [n_sample]: the sample densities rho_i */
} aqr_train_cfg;

/* Encode n base vectors x (device [n x d] fp32, row stride ld_x >= d floats) into codes
 * (device [n x qp->d_pad] u8; padding bytes are written as 0):
 *     code_ij = roundf(clamp((x_ij - min_j) * scale_j, 0, 255))   (fp32; Alg1 l.9; R5)
 * If `train` is non-NULL the quantizer is first trained on x (density kNN over the sample in
 * fp64 -> delta -> per-dimension linear percentiles over all n points -> min/max/scale) and
 * the stream is synchronized before returning (delta etc. are returned on the host).
 * If `train` is NULL, qp must hold trained parameters and the call is asynchronous.
 * Temporary device memory for training (n*d*4 bytes) is allocated stream-ordered inside. */
aqr_status aqr_encode(const float *x, int64_t n, int32_t d, int64_t ld_x, const aqr_train_cfg *train,
                      aqr_quant_params *qp, uint8_t *codes, aqr_stream_t stream);

/* ------------------------------------------------------------------------------------ */
/* aqr_upload_index -- the HNSW graph + codes + fp32 vectors (Alg1 l.16-22)    */
/* ------------------------------------------------------------------------------------ */

typedef struct aqr_index aqr_index; /* opaque, library-owned, immutable after upload */

typedef struct {
  int64_t n;                 /* number of base vectors, 1 <= n < 2^31 */
  int32_t d;                 /* dimensionality */
  aqr_metric metric;         /* AQR_L2 or AQR_IP (R12: stages 2-3 use 1 - <q,x>) */
  int64_t id_base;           /* added to every returned id (shard offset for C5) */
  const uint8_t *codes;      /* device [n x d_pad] from aqr_encode */
  int32_t d_pad;             /* code row stride (multiple of 16, >= d) */
  const float *base;         /* device [n x ld_base] fp32 vectors kept for re-rank (Alg1 l.21) */
  int64_t ld_base;           /* >= d */
  const float *min_j;        /* device [d] trained quantizer (aqr_quant_params) */
  const float *scale_j;      /* device [d] */
  int32_t M;                 /* degree cap at layers >= 1 (1..80); layer-0 rows hold 2*M entries */
  int32_t max_level;         /* top layer */
  int32_t entry_point;       /* a node of level max_level */
  const int32_t *adj0;       /* host [n x 2M], -1 padded, ids in [0, n) */
  const int64_t *upper_off;  /* host [n]: row in adj_upper of (node, layer 1), -1 for level-0 nodes;
                                layer L (1 <= L <= level) of node v is row upper_off[v] + L - 1 */
  const int32_t *adj_upper;  /* host [upper_rows x M], -1 padded (may be NULL if upper_rows == 0) */
  int64_t upper_rows;
  int32_t layout;            /* AQR_LAYOUT_AUTO / _GATHER / _INLINE (see below) */
} aqr_index_desc;

/* Layer-0 layout of the uploaded index.
 *  GATHER: adjacency rows [n x 2M] int32 and the code array [n x d_pad]; an expansion reads
 *          the row, then gathers one code row per neighbour (two dependent DRAM round trips).
 *  INLINE: one contiguous block per node = its layer-0 neighbour ids followed by the codes of
 *          those neighbours (n x 2M x d_pad bytes, ~7 GB for 1M x 128 at M = 27); an expansion
 *          is ONE bulk (TMA) copy of that block into shared memory, prefetched while the
 *          previous expansion's merge runs.  Uses HBM capacity to remove a round trip.
 *  AUTO:   GATHER (measured faster on B200 at every C2 ef point, profiles/r01).
 * Both layouts give identical results (same visit order, same ids). */
enum { AQR_LAYOUT_AUTO = 0, AQR_LAYOUT_GATHER = 1, AQR_LAYOUT_INLINE = 2 };

/* Copy the index into library-owned device buffers re-laid-out for the search kernel
 * (code rows padded with zeros to a multiple of 32 bytes, one 256-bit load per 32 bytes, fp32 rows padded to a multiple of 4 floats, layer-0 rows padded
 * to a multiple of 8 entries).  The caller may free its inputs once the stream is
 * synchronized (this call synchronizes the stream before returning).  Validates ids,
 * entry point and sizes, and rejects a row (layer 0 or upper) that lists a neighbour twice or
 * lists its own node (AQR_E_INVALID): the beam keeps no visited set by default (R15),
 * so a repeated id would be scored twice in one expansion and enter W twice. */
aqr_status aqr_upload_index(const aqr_index_desc *desc, aqr_index **out, aqr_stream_t stream);
void aqr_index_free(aqr_index *ix);
/* bytes of device memory owned by the index */
size_t aqr_index_device_bytes(const aqr_index *ix);
/* the layout chosen at upload (AQR_LAYOUT_GATHER or AQR_LAYOUT_INLINE) */
int32_t aqr_index_layout(const aqr_index *ix);

/* ------------------------------------------------------------------------------------ */
/* aqr_search -- Alg2 fused: quantize query, Stage 1 (greedy upper layers + layer-0 beam on */
/* d^q), Stage 2 (asymmetric d^a), early termination, Stage 3 (exact d^e), assembly.      */
/* ------------------------------------------------------------------------------------ */

typedef struct {
  int32_t k;            /* results per query (Alg2 l.1) */
  int32_t ef;           /* layer-0 beam width ef_search (N_c x m_ef, R13), <= 8192 */
  int32_t n_coarse;     /* N_c: |C| handed to Stage 2; k <= n_coarse <= ef */
  int32_t n_rerank;     /* N_rerank: exact re-rank depth (Alg2 l.20); 0 <= n_rerank <= n_coarse */
  double tau_gap;       /* >= 0 */
  double tau_ratio;     /* >= 1 */
  int32_t early_term;   /* 1 = apply the early-termination test (Alg2 l.15-16) */
  int32_t assemble_mode;/* 0 = fill (R10, default), 1 = union */
  int32_t visited_bits; /* GATHER layout: log2 of the per-query visited-hash slots in shared memory,
                           6..16; 0 or -1 = no visited set (default): re-encountered nodes are
                           re-scored and dropped by the W dedupe (R15); -2 = exact visited bitmap
                           in global memory (one n-bit map per warp slot, in the caller's workspace:
                           size it with aqr_search_workspace_size), no shared memory.  Results are
                           identical in every mode.  INLINE layout (AQR traversal): only 0 / -1;
                           -2 and 6..16 are rejected (AQR_E_INVALID): that beam keeps no visited set. */
  int32_t warps_per_block; /* reserved, must be 0 (the CTA shape is fixed at compile time) */
  int32_t traversal;    /* AQR_TRAVERSAL_AQR (0): the method (Alg2).  AQR_TRAVERSAL_FP32 (1): the
                           paper's baseline (plain HNSW search) on the same graph: greedy
                           descent and the layer-0 beam on exact fp32 distances (L2, or 1 - <q,x>),
                           result = the first k of W; n_coarse bounds the traced C, n_rerank /
                           early_term / assemble_mode are ignored.  GATHER kernels only (an INLINE
                           index is searched through its GATHER arrays). */
  double tau_spread;    /* adaptive re-rank depth ("evaluates the spread of asymmetric
                           distances", R27): >= 0 re-ranks only the entries of A with
                           d^a <= (1 + tau_spread) d^a_k (at least k, at most n_rerank); +inf
                           (INFINITY) = the static n_rerank.  NaN or < 0: AQR_E_INVALID. */
  int32_t warps_per_query; /* 0 = auto (default), 1 = one warp per query, 4 = one CTA of 4 warps per
                           query: the warps split each expansion's visited test, code gathers,
                           scoring, W dedupe and W insert (same results, visit order and counters).
                           Auto picks 4 for GATHER-layout AQR searches whose one-warp launch holds
                           <= 4 queries per SM (large ef: W alone fills the shared memory).  4 with the FP32 traversal or an INLINE index (AQR traversal):
                           AQR_E_INVALID; other values: AQR_E_INVALID. */
} aqr_search_params;

enum { AQR_TRAVERSAL_AQR = 0, AQR_TRAVERSAL_FP32 = 1 };

#define AQR_NCOUNT 15
/* counter slots: 0 expansions, 1 layer-0 degree sum, 2 layer-0 code evaluations, 3 upper
 * expansions, 4 upper degree sum, 5 upper evaluations, 6 |C|, 7 re-rank depth, 8 early-term
 * flag, 9 |A|, 10 visited-hash insert failures (re-evaluations allowed by DESIGN.md R15),
 * 11 evaluations below the W threshold, 12 W insertions (11 minus re-evaluations already in
 * W) (kernel bookkeeping; no oracle counterpart), 13-14 reserved (0) */

/* Optional transcript (all device pointers, each may be NULL).  Per-query arrays are laid
 * out [nq x ...].  Used by the parity tests to compare visit order with the oracle. */
typedef struct {
  int32_t exp_cap;      /* capacity of each exp_ids row */
  int32_t *exp_ids;     /* [nq x exp_cap] layer-0 expansion sequence */
  int32_t *coarse_ids;  /* [nq x n_coarse] C in (d^q, id) order */
  int32_t *coarse_dq;   /* [nq x n_coarse] d^q of C (integer, s_dist not applied) */
  int32_t *asym_ids;    /* [nq x n_coarse] A in (d^a, id) order */
  float *asym_d;        /* [nq x n_coarse] d^a */
  float *exact_d;       /* [nq x n_coarse] d^e of A[0:depth] */
  int64_t *counters;    /* [nq x AQR_NCOUNT] */
  int64_t *totals;      /* [AQR_NCOUNT] summed over queries (atomic adds) */
  int64_t *t_ns;        /* [nq x 2] %globaltimer (ns) when a warp took the query and when its
                           outputs were written: per-query latency inside a batch (Fig. 4).
                           Timing alone (all other pointers NULL) adds no trace work. */
} aqr_debug;

/* Bytes of caller workspace aqr_search needs (device, any alignment >= 16): 256, plus, for
 * visited_bits = -2, min(nq rounded up to 4, 64 x SMs) bitmaps of ceil(n / 128) x 16 bytes. */
size_t aqr_search_workspace_size(const aqr_index *ix, int64_t nq, const aqr_search_params *p);

/* Search nq queries q (device [nq x ld_q] fp32).  Writes out_ids (device [nq x k] int32,
 * id_base + node id, -1 padding) and out_dist (device [nq x k] fp32: d^e for re-ranked
 * entries, d^a for entries filled from A; +inf padding), sorted by (dist, id).
 * One warp (or one CTA of 4 warps, warps_per_query) per query, persistent grid; asynchronous
 * on `stream`. */
aqr_status aqr_search(const aqr_index *ix, const float *q, int64_t nq, int64_t ld_q,
                      const aqr_search_params *p, int32_t *out_ids, float *out_dist,
                      const aqr_debug *debug, void *ws, size_t ws_bytes, aqr_stream_t stream);

/* The launch aqr_search would make for these arguments, without launching: *warps_per_query =
 * 1 (one warp per query) or 4 (one cooperative CTA of 4 warps per query), resolving
 * p->warps_per_query = 0 (auto) by the rule above.  Host-only (an occupancy query on the current
 * device); validation as aqr_search. */
aqr_status aqr_search_plan(const aqr_index *ix, int64_t nq, const aqr_search_params *p,
                           int32_t *warps_per_query);

/* Stages 2 / ET / 3 / assembly alone (Alg2 l.8-24) on caller-supplied coarse lists:
 * cand_ids device [nq x n_cand] int32 node ids sorted by (d^q, id); a -1 ends a list early.
 * p->k, n_rerank, tau_*, early_term, assemble_mode are used (n_coarse := n_cand). */
aqr_status aqr_rerank(const aqr_index *ix, const float *q, int64_t nq, int64_t ld_q,
                      const int32_t *cand_ids, int32_t n_cand, const aqr_search_params *p,
                      int32_t *out_ids, float *out_dist, aqr_stream_t stream);

/* Merge n_lists per-shard result lists (device dist/ids [n_lists x nq x k], each row sorted
 * by (dist, id), -1 ids = padding) into the global top-k by (dist, id) (BJ configs[4]). */
aqr_status aqr_merge_topk(const float *dist, const int32_t *ids, int32_t n_lists, int64_t nq,
                          int32_t k, float *out_dist, int32_t *out_ids, aqr_stream_t stream);

/* ------------------------------------------------------------------------------------ */
/* Peer-memory exchange for the sharded configuration (BASELINE.json configs[4]: "per-shard  */
/* top-k gathered over NVLink and merged"; SURVEY 8(e) fused variant).  One process per GPU. */
/* Each rank owns a block of the query batch.  A rank searches every query on its shard(s)    */
/* with aqr_search, one launch per destination block, with out_ids / out_dist pointing INTO    */
/* the owner's gather buffer (a peer-mapped pointer; the owner's own block is a local one):    */
/* the search kernel's epilogue stores are the NVLink transfer.  Then aqr_peer_signal, on the  */
/* owner aqr_peer_wait, and aqr_merge_topk over the [n_lists x blk x k] lists of its block.    */
/* No NCCL call on the data path.                                                              */
/* ------------------------------------------------------------------------------------ */
#define AQR_MAX_PEERS 8
#define AQR_PEER_HANDLE_BYTES 64

/* cudaMalloc `bytes` (zero-filled) on the current device and export it: *dptr the local device
 * pointer, handle[64] an IPC handle another process on this node opens with aqr_peer_open.
 * Errors: AQR_E_INVALID, AQR_E_OOM, AQR_E_CUDA.  Free with aqr_peer_free (after every peer closed it). */
aqr_status aqr_peer_alloc(size_t bytes, void **dptr, uint8_t *handle);
/* Map a peer process's allocation (handle from ITS aqr_peer_alloc) into this process: *dptr is
 * valid on the current device (peer access over NVLink is enabled by the mapping).  A process
 * must not open its own handle (use the local pointer).  Unmap with aqr_peer_close. */
aqr_status aqr_peer_open(const uint8_t *handle, void **dptr);
aqr_status aqr_peer_close(void *dptr);
aqr_status aqr_peer_free(void *dptr);
/* After every kernel launched on `stream` so far: flags[i][slot] = value for i < n_peers, with
 * system-scope release semantics (the stores those kernels made to peer memory are visible to a
 * peer that acquires the flag).  flags: HOST array of n_peers DEVICE pointers (peer-mapped, or
 * local for this rank's own) to uint64 arrays; 1 <= n_peers <= AQR_MAX_PEERS; value must grow
 * from step to step.  Asynchronous. */
aqr_status aqr_peer_signal(uint64_t *const *flags, int32_t n_peers, int32_t slot, uint64_t value,
                           aqr_stream_t stream);
/* Block `stream` (a spinning kernel, system-scope acquire loads) until flags[i] >= value for every
 * i < n (flags: LOCAL device array, 1 <= n <= 32).  A flag still below value after timeout_ns
 * makes the kernel give up and write 1 + i to *status (device int32, zeroed by the caller; may be
 * NULL): the caller checks it after synchronizing.  Asynchronous. */
aqr_status aqr_peer_wait(const uint64_t *flags, int32_t n, uint64_t value, uint64_t timeout_ns,
                         int32_t *status, aqr_stream_t stream);

/* Thread-local description of the last failure ("" if none). */
const char *aqr_last_error(void);
/* ------------------------------------------------------------------------------------ */
/* aqr_build_graph -- the index build, Alg1 Stage 3 (G.Insert(q_i, i, M_i, ef^c) */
/* for i = 1..n) on the GPU: HNSW insertion [23] over the quantized     */
/* codes with the integer distance d^q and (d, id) ties, Malkov's neighbour heuristic        */
/* (R14), nodes inserted in id order in waves (R28).  The result is byte-identical */
/* to the oracle's or_build_graph and the host builder for the same inputs.                  */
/* ------------------------------------------------------------------------------------ */
/* codes:      device [n x d_pad] u8 (aqr_encode's layout, d_pad = round_up(d, 16))
 * levels:     host [n], each in [0, 30] (floor(-ln(u) / ln(M)) from seeded draws)
 * upper_off:  host [n]: row of (v, layer 1), rows of a node consecutive, -1 iff levels[v] = 0;
 *             upper_rows = sum of levels
 * M:          degree cap at layers >= 1 (2..80); layer-0 rows hold 2M (M_i of Alg1 l.17)
 * efc:        ef^construction (Alg1 l.18), 1..1024
 * flags:      bit 0 keepPrunedConnections (R14); bit 1 a new node selects 2M layer-0 neighbours
 * batch_div:  wave size = min(max(1, pos / batch_div), 4096) (0 = 32; R28)
 * adj0:       host out [n x 2M], -1 padded;  adj_upper: host out [upper_rows x M], -1 padded
 * entry_max:  host out {entry point, top level}
 * Device memory is allocated and released inside (about n x (d_pad + 8 M + 12) bytes plus a
 * few hundred MB of wave scratch).  Synchronous: returns when the host arrays are filled.
 * Errors: AQR_E_INVALID (arguments), AQR_E_OOM, AQR_E_CUDA. */
aqr_status aqr_build_graph(const uint8_t *codes, int64_t n, int32_t d, int32_t d_pad, const int32_t *levels,
                           const int64_t *upper_off, int64_t upper_rows, int32_t M, int32_t efc, int32_t flags,
                           int32_t batch_div, int32_t *adj0, int32_t *adj_upper, int32_t *entry_max,
                           aqr_stream_t stream);

/* "aqr-b200 <version> (sm_100a) src:<16 hex digits>": the hash of the CUDA sources this
 * library was compiled from (build.py rebuilds when it differs from the sources in the tree). */
const char *aqr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AQR_H_ */
