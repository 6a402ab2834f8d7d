/*
 * aqr_oracle.c -- plain, slow, single-threaded CPU ORACLE for the AQR-HNSW hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2602_21600_b200/csrc) and includes nothing
 * from it.  Compiled with  gcc -O2 -ffp-contract=off -fno-fast-math  (no FMA contraction;
 * fmaf() is called explicitly where the paper says FMA).
 *
 * Citations: P:n = /root/reference/PAPER.md line n, "Alg1 l.k" / "Alg2 l.k" = the
 * algorithm's own line (its PAPER.md line is given too), S:n = SPEC.md line n,
 * DESIGN.md R<n> = a reading of the paper recorded in DESIGN.md "Readings".
 *
 * Every function is the paper's definition written out in the paper's order; a library
 * primitive (qsort) serves as the sort step.  No blocking, fusion or reordering.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): see DESIGN.md "Oracle pins".  Functions
 * without an independent pin: none (recall values on synthetic data are "parity unpinned"
 * -- they are measurements, not oracle functions).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENOMEM 3

/* ------------------------------------------------------------------------------------ */
/* sorting helpers (qsort is the library primitive; comparators implement the (value,id) */
/* total order used everywhere, "ties broken by ascending id")                     */
/* ------------------------------------------------------------------------------------ */
typedef struct { double v; int64_t id; } or_dpair;
typedef struct { float v; int32_t id; } or_fpair;

static int cmp_dpair(const void *a, const void *b) {
  const or_dpair *x = (const or_dpair *)a, *y = (const or_dpair *)b;
  if (x->v < y->v) return -1;
  if (x->v > y->v) return 1;
  return (x->id < y->id) ? -1 : (x->id > y->id);
}
static int cmp_fpair(const void *a, const void *b) {
  const or_fpair *x = (const or_fpair *)a, *y = (const or_fpair *)b;
  if (x->v < y->v) return -1;
  if (x->v > y->v) return 1;
  return (x->id < y->id) ? -1 : (x->id > y->id);
}
static int cmp_double(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return (x < y) ? -1 : (x > y);
}

/* ==================================================================================== */
/* Build phase, Stage 1: density characterisation (Alg1 l.5-6 at P:114-115)     */
/* ==================================================================================== */

/* rho_i = 1 / (dbar_k(x_i) + eps), dbar_k = (1/k) sum over the k nearest neighbours of the
 * SQUARED L2 distance.  kNN is taken within the sample, self excluded, ties
 * by id.  fp64: diff = (double)x_it - (double)x_jt; acc = acc + diff*diff (t ascending).
 * The k smallest are summed in ascending (value,id) order, then divided by k. */
int or_density(const float *x, int64_t n, int32_t d, const int32_t *sample, int32_t ns,
               int32_t k, double eps, double *rho_out) {
  if (!x || !sample || !rho_out || n < 1 || d < 1 || ns < 1 || k < 1 || ns <= k) return OR_EINVAL;
  or_dpair *dist = (or_dpair *)malloc(sizeof(or_dpair) * (size_t)ns);
  if (!dist) return OR_ENOMEM;
  for (int32_t a = 0; a < ns; ++a) {
    const float *xi = x + (int64_t)sample[a] * d;
    int32_t m = 0;
    for (int32_t b = 0; b < ns; ++b) {
      if (b == a) continue;
      const float *xj = x + (int64_t)sample[b] * d;
      double acc = 0.0;
      for (int32_t t = 0; t < d; ++t) {
        double diff = (double)xi[t] - (double)xj[t];
        acc = acc + diff * diff;
      }
      dist[m].v = acc;
      dist[m].id = sample[b];
      ++m;
    }
    qsort(dist, (size_t)m, sizeof(or_dpair), cmp_dpair);
    double s = 0.0;
    for (int32_t t = 0; t < k; ++t) s = s + dist[t].v;
    double mean = s / (double)k;
    rho_out[a] = 1.0 / (mean + eps);
  }
  free(dist);
  return OR_OK;
}

/* delta = (max_i rho_i - min_i rho_i) / (max_i rho_i + eps)   (Alg1 l.6) */
double or_delta(const double *rho, int32_t ns, double eps) {
  double mx = rho[0], mn = rho[0];
  for (int32_t i = 1; i < ns; ++i) {
    if (rho[i] > mx) mx = rho[i];
    if (rho[i] < mn) mn = rho[i];
  }
  return (mx - mn) / (mx + eps);
}

/* ==================================================================================== */
/* Build phase, Stage 2: quantizer training (Alg1 l.8-11 at P:117-120)           */
/* ==================================================================================== */

/* Linear-interpolated percentile P (percent scale, R3/R4) of an ascending array
 * s[0..n-1]:  r = (P/100)(n-1); lo = floor(r); hi = min(lo+1, n-1); f = r - lo;
 * v = s[lo] + f*(s[hi]-s[lo])  (numpy "linear"; separate mul and add). */
double or_percentile_sorted(const double *s, int64_t n, double P) {
  double r = (P / 100.0) * (double)(n - 1);
  int64_t lo = (int64_t)floor(r);
  if (lo < 0) lo = 0;
  if (lo > n - 1) lo = n - 1;
  int64_t hi = (lo + 1 < n - 1) ? lo + 1 : n - 1;
  double f = r - (double)lo;
  double diff = s[hi] - s[lo];
  double prod = f * diff;
  return s[lo] + prod;
}

/* Train the per-dimension quantizer.
 *   P_l = delta * P_max, P_h = 100 - delta * P_max   (Alg1 l.8 at P:117, percent scale R3)
 *   min_j = P_l-percentile of column j over ALL n points, max_j = P_h-percentile
 *   scale_j = 255 / (max_j - min_j + eps)           (Alg1 l.11 at P:120)
 *   degenerate range (< 1e-9): scale_j = 1 (R6)
 * Outputs are rounded once to fp32.  meta = {delta, P_l, P_h}.
 * delta: if delta_override is not NaN it is used, else computed from the sample (O1-O3). */
int or_train(const float *x, int64_t n, int32_t d, const int32_t *sample, int32_t ns,
             int32_t k_density, double p_max, double delta_override, double eps,
             float *min_f, float *max_f, float *scale_f, double *meta) {
  if (!x || n < 1 || d < 1 || !min_f || !max_f || !scale_f || !meta) return OR_EINVAL;
  double delta;
  if (!isnan(delta_override)) {
    delta = delta_override;
  } else {
    double *rho = (double *)malloc(sizeof(double) * (size_t)ns);
    if (!rho) return OR_ENOMEM;
    int st = or_density(x, n, d, sample, ns, k_density, eps, rho);
    if (st) { free(rho); return st; }
    delta = or_delta(rho, ns, eps);
    free(rho);
  }
  double p_l = delta * p_max;
  double p_h = 100.0 - delta * p_max;
  double *col = (double *)malloc(sizeof(double) * (size_t)n);
  if (!col) return OR_ENOMEM;
  for (int32_t j = 0; j < d; ++j) {
    for (int64_t i = 0; i < n; ++i) col[i] = (double)x[i * d + j];
    qsort(col, (size_t)n, sizeof(double), cmp_double);
    double mn = or_percentile_sorted(col, n, p_l);
    double mx = or_percentile_sorted(col, n, p_h);
    double range = mx - mn;
    min_f[j] = (float)mn;
    max_f[j] = (float)mx;
    if (range < 1e-9) {
      scale_f[j] = 1.0f;
    } else {
      scale_f[j] = (float)(255.0 / (range + eps));
    }
  }
  free(col);
  meta[0] = delta;
  meta[1] = p_l;
  meta[2] = p_h;
  return OR_OK;
}

/* Quantize (Alg1 l.9 at P:118; "shifted and scaled into the 0-255 range, clipped ...,
 * then rounded to the nearest integer"; query: Alg2 l.4 at P:165).  fp32 arithmetic:
 * t = x - min; u = t * scale; v = clamp(u, 0, 255); code = roundf(v) (half away, R5).
 * Rows are written with stride d_pad; bytes d..d_pad-1 are zero. */
void or_encode(const float *x, int64_t n, int32_t d, const float *min_f, const float *scale_f,
               uint8_t *codes, int32_t d_pad) {
  for (int64_t i = 0; i < n; ++i) {
    for (int32_t j = 0; j < d; ++j) {
      float t = x[i * d + j] - min_f[j];
      float u = t * scale_f[j];
      float v = u;
      if (v < 0.0f) v = 0.0f;
      if (v > 255.0f) v = 255.0f;
      codes[i * d_pad + j] = (uint8_t)roundf(v);
    }
    for (int32_t j = d; j < d_pad; ++j) codes[i * d_pad + j] = 0;
  }
}

/* ==================================================================================== */
/* Search phase (Alg2)                                                        */
/* ==================================================================================== */

typedef struct {
  int64_t n;
  int32_t d, d_pad, metric;       /* metric 0 = L2, 1 = inner product (R12) */
  const uint8_t *codes;           /* [n x d_pad] */
  const float *base;              /* [n x d] fp32, kept for re-rank (Alg1 l.21) */
  const float *min_f, *scale_f;   /* [d] */
  int32_t max_level, entry_point;
  int32_t cap0;                   /* layer-0 row width (2M), -1 padded */
  const int32_t *adj0;            /* [n x cap0] */
  int32_t capu;                   /* layer>=1 row width (M), -1 padded */
  const int64_t *upper_off;       /* [n]: row of (node, layer 1) in adj_upper, -1 if level 0 */
  const int32_t *adj_upper;       /* rows of width capu; layer L of node v is row upper_off[v]+L-1 */
  const int32_t *levels;          /* [n] */
} or_index;

typedef struct {
  int32_t k, ef, n_coarse, n_rerank;
  double tau_gap, tau_ratio;
  int32_t early_term, assemble_mode; /* 0 = fill (R10), 1 = union */
  int32_t beam_form;                 /* 0 = flag form (R8), 1 = Malkov heap form */
  int32_t traversal;                 /* 0 = AQR (Alg2), 1 = FP32-HNSW baseline */
  double tau_spread;                 /* adaptive re-rank depth (R27): +inf = the
                                        static N_rerank; else depth = the entries of A with
                                        d^a <= (1 + tau_spread) d^a_k, at least k, at most N_rerank */
} or_params;

/* per-query trace; any pointer may be NULL */
typedef struct {
  int32_t exp_cap;
  int32_t *exp_ids;       /* layer-0 expansion sequence (visit order) */
  int32_t *coarse_ids;    /* [n_coarse]  C (Alg2 l.7) */
  int32_t *coarse_dq;     /* [n_coarse]  d^q of C */
  int32_t *asym_ids;      /* [n_coarse]  A (Alg2 l.13) */
  float *asym_d;          /* [n_coarse]  d^a of A */
  float *exact_d;         /* [n_coarse]  d^e of A[0:depth] */
  int64_t *counters;      /* [OR_NCOUNT] */
  int32_t upper_cap;      /* entries of upper_end (>= max_level to record every layer) */
  int32_t *upper_end;     /* [upper_cap] node where the descent leaves layer L, stored at
                             index max_level - L (trace only: no arithmetic depends on it) */
} or_trace;

enum {
  C_EXPANSIONS = 0, C_DEG_SUM, C_EVALS, C_UPPER_EXP, C_UPPER_DEG_SUM, C_UPPER_EVALS,
  C_NC, C_DEPTH, C_ET, C_NA, OR_NCOUNT
};

/* Quantized distance d^q = sum_j (qhat_j - xhat_j)^2 as an integer (Alg2 l.6).
 * s_dist is a positive constant factor and is not applied (ordering-invariant, R7).  */
static int32_t dq_dist(const uint8_t *qc, const uint8_t *xc, int32_t d) {
  int32_t s = 0;
  for (int32_t j = 0; j < d; ++j) {
    int32_t e = (int32_t)qc[j] - (int32_t)xc[j];
    s += e * e;
  }
  return s;
}

static int key_less(int32_t da, int32_t ia, int32_t db, int32_t ib) {
  return (da < db) || (da == db && ia < ib);
}

static const int32_t *nbr_row(const or_index *ix, int32_t v, int32_t layer, int32_t *cap) {
  if (layer == 0) { *cap = ix->cap0; return ix->adj0 + (int64_t)v * ix->cap0; }
  *cap = ix->capu;
  return ix->adj_upper + (ix->upper_off[v] + layer - 1) * ix->capu;
}

/* Greedy descent through layers max_level..1 ("greedily traverses"; R8):
 * repeat cur <- argmin over {cur} U N_L(cur) of (d^q, id) until it stops changing. */
static int32_t greedy(const or_index *ix, const uint8_t *qc, int32_t *dcur_out, int64_t *cnt,
                      or_trace *tr) {
  int32_t cur = ix->entry_point;
  int32_t dcur = dq_dist(qc, ix->codes + (int64_t)cur * ix->d_pad, ix->d);
  if (cnt) cnt[C_UPPER_EVALS] += 1;
  for (int32_t L = ix->max_level; L >= 1; --L) {
    for (;;) {
      int32_t cap;
      const int32_t *row = nbr_row(ix, cur, L, &cap);
      int32_t best = cur, dbest = dcur, deg = 0;
      for (int32_t t = 0; t < cap; ++t) {
        int32_t u = row[t];
        if (u < 0) continue;
        ++deg;
        int32_t du = dq_dist(qc, ix->codes + (int64_t)u * ix->d_pad, ix->d);
        if (cnt) cnt[C_UPPER_EVALS] += 1;
        if (key_less(du, u, dbest, best)) { best = u; dbest = du; }
      }
      if (cnt) { cnt[C_UPPER_EXP] += 1; cnt[C_UPPER_DEG_SUM] += deg; }
      if (best == cur) break;
      cur = best;
      dcur = dbest;
    }
    if (tr && tr->upper_end && ix->max_level - L < tr->upper_cap) tr->upper_end[ix->max_level - L] = cur;
  }
  *dcur_out = dcur;
  return cur;
}

/* W: sorted bounded list of (d^q, id, expanded) -- the "flag form" of the layer-0 beam
 * (R8).  Returns |W|; W holds the final list. */
typedef struct { int32_t d, id; uint8_t expanded; } or_went;

static int32_t beam_flag(const or_index *ix, const uint8_t *qc, int32_t ep, int32_t dep,
                         int32_t ef, uint8_t *visited, or_went *W, or_trace *tr) {
  int32_t size = 1;
  W[0].d = dep; W[0].id = ep; W[0].expanded = 0;
  visited[ep] = 1;
  int32_t nexp = 0;
  for (;;) {
    int32_t ci = -1;
    for (int32_t i = 0; i < size; ++i)
      if (!W[i].expanded) { ci = i; break; }
    if (ci < 0) break;
    W[ci].expanded = 1;
    int32_t c = W[ci].id;
    if (tr && tr->exp_ids && nexp < tr->exp_cap) tr->exp_ids[nexp] = c;
    ++nexp;
    int32_t cap;
    const int32_t *row = nbr_row(ix, c, 0, &cap);
    int32_t deg = 0;
    for (int32_t t = 0; t < cap; ++t) {
      int32_t u = row[t];
      if (u < 0) continue;
      ++deg;
      if (visited[u]) continue;
      visited[u] = 1;
      int32_t du = dq_dist(qc, ix->codes + (int64_t)u * ix->d_pad, ix->d);
      if (tr && tr->counters) tr->counters[C_EVALS] += 1;
      if (size < ef || key_less(du, u, W[size - 1].d, W[size - 1].id)) {
        int32_t pos = size < ef ? size : ef - 1;  /* slot freed (or evicted last) */
        while (pos > 0 && key_less(du, u, W[pos - 1].d, W[pos - 1].id)) {
          W[pos] = W[pos - 1];
          --pos;
        }
        W[pos].d = du; W[pos].id = u; W[pos].expanded = 0;
        if (size < ef) ++size;
      }
    }
    if (tr && tr->counters) tr->counters[C_DEG_SUM] += deg;
  }
  if (tr && tr->counters) tr->counters[C_EXPANSIONS] += nexp;
  return size;
}

/* Malkov's SEARCH-LAYER (heap form), written with plain arrays: candidate set C (min by
 * (d,id)), result set W (max by (d,id)), stop when min C > max W.  Used to cross-check the
 * flag form. */
static int32_t beam_heap(const or_index *ix, const uint8_t *qc, int32_t ep, int32_t dep,
                         int32_t ef, uint8_t *visited, or_went *W, or_trace *tr) {
  int64_t ccap = 1024, csz = 0;
  or_went *C = (or_went *)malloc(sizeof(or_went) * (size_t)ccap);
  int32_t wsz = 0;
  or_went *R = (or_went *)malloc(sizeof(or_went) * (size_t)(ef + 1));
  C[csz].d = dep; C[csz].id = ep; ++csz;
  R[wsz].d = dep; R[wsz].id = ep; ++wsz;
  visited[ep] = 1;
  int32_t nexp = 0;
  while (csz > 0) {
    int64_t mi = 0;
    for (int64_t i = 1; i < csz; ++i)
      if (key_less(C[i].d, C[i].id, C[mi].d, C[mi].id)) mi = i;
    or_went c = C[mi];
    C[mi] = C[csz - 1];
    --csz;
    int32_t fi = 0;
    for (int32_t i = 1; i < wsz; ++i)
      if (key_less(R[fi].d, R[fi].id, R[i].d, R[i].id)) fi = i;
    if (key_less(R[fi].d, R[fi].id, c.d, c.id)) break;
    if (tr && tr->exp_ids && nexp < tr->exp_cap) tr->exp_ids[nexp] = c.id;
    ++nexp;
    int32_t cap;
    const int32_t *row = nbr_row(ix, c.id, 0, &cap);
    for (int32_t t = 0; t < cap; ++t) {
      int32_t u = row[t];
      if (u < 0 || visited[u]) continue;
      visited[u] = 1;
      int32_t du = dq_dist(qc, ix->codes + (int64_t)u * ix->d_pad, ix->d);
      fi = 0;
      for (int32_t i = 1; i < wsz; ++i)
        if (key_less(R[fi].d, R[fi].id, R[i].d, R[i].id)) fi = i;
      if (wsz < ef || key_less(du, u, R[fi].d, R[fi].id)) {
        if (csz == ccap) { ccap *= 2; C = (or_went *)realloc(C, sizeof(or_went) * (size_t)ccap); }
        C[csz].d = du; C[csz].id = u; ++csz;
        R[wsz].d = du; R[wsz].id = u; ++wsz;
        if (wsz > ef) {
          fi = 0;
          for (int32_t i = 1; i < wsz; ++i)
            if (key_less(R[fi].d, R[fi].id, R[i].d, R[i].id)) fi = i;
          R[fi] = R[wsz - 1];
          --wsz;
        }
      }
    }
  }
  /* sort the result set ascending by (d, id) */
  for (int32_t i = 1; i < wsz; ++i) {
    or_went e = R[i];
    int32_t p = i;
    while (p > 0 && key_less(e.d, e.id, R[p - 1].d, R[p - 1].id)) { R[p] = R[p - 1]; --p; }
    R[p] = e;
  }
  for (int32_t i = 0; i < wsz; ++i) { W[i] = R[i]; W[i].expanded = 1; }
  free(C);
  free(R);
  return wsz;
}

/* Stage 2 decode (Alg2 l.11): x~_j = xhat_j / scale_j + min_j (fp32 division, R9). */
static float decode_elem(uint8_t c, float scale, float mn) {
  float v = (float)c / scale;
  return v + mn;
}

/* The fp32 sums of Stages 2 and 3 are taken in the canonical order R(32) of SURVEY 8(c)
 * (O11/O13, "Canonical fp32 reduction R(L)"): element j belongs to the 4-wide chunk t = j/4,
 * chunk t to partial l = t mod 32; partial l starts at +0 and accumulates its terms with one FMA
 * each, chunks in increasing t and elements in increasing j; then, for off = 16 .. 1,
 * every partial becomes p[l] + p[l ^ off]; the result is p[0].  A summation order is a choice
 * the paper leaves open (it only says "FMA"); fixing it makes the fp32 values
 * reproducible bit for bit, so no 1-ulp difference can flip the re-rank cut, the ET test or a
 * tie by id.  tests/test_oracle_pins.py bounds it against an fp64 sum (north_star: 1e-5). */
static float butterfly32(float *p) {
  float t2[32];
  for (int32_t off = 16; off >= 1; off /= 2) {
    for (int32_t l = 0; l < 32; ++l) t2[l] = p[l] + p[l ^ off];
    for (int32_t l = 0; l < 32; ++l) p[l] = t2[l];
  }
  return p[0];
}

/* d^a (Alg2 l.9): sum_j (q_j - x~_j)^2, an FMA per term, order R(32).
 * Inner product (R12): 1 - sum_j q_j x~_j. */
static float asym_dist(const or_index *ix, const float *q, const uint8_t *xc) {
  float p[32];
  for (int32_t l = 0; l < 32; ++l) p[l] = 0.0f;
  for (int32_t j = 0; j < ix->d; ++j) {
    float xt = decode_elem(xc[j], ix->scale_f[j], ix->min_f[j]);
    int32_t l = (j / 4) % 32;
    if (ix->metric == 0) {
      float e = q[j] - xt;
      p[l] = fmaf(e, e, p[l]);
    } else {
      p[l] = fmaf(q[j], xt, p[l]);
    }
  }
  float acc = butterfly32(p);
  return ix->metric == 0 ? acc : 1.0f - acc;
}

/* d^e (Alg2 l.19; P:197 FMA): sum_j (q_j - x_j)^2 in order R(32); IP: 1 - q.x */
static float exact_dist(const or_index *ix, const float *q, const float *x) {
  float p[32];
  for (int32_t l = 0; l < 32; ++l) p[l] = 0.0f;
  for (int32_t j = 0; j < ix->d; ++j) {
    int32_t l = (j / 4) % 32;
    if (ix->metric == 0) {
      float e = q[j] - x[j];
      p[l] = fmaf(e, e, p[l]);
    } else {
      p[l] = fmaf(q[j], x[j], p[l]);
    }
  }
  float acc = butterfly32(p);
  return ix->metric == 0 ? acc : 1.0f - acc;
}

/* Stages 2, ET, 3 and assembly for one query given C (ids sorted by (d^q,id)).
 * Alg2 l.8-24.  Writes k results (padded with -1 / +inf). */
static int rerank_one(const or_index *ix, const float *q, const int32_t *cids, int32_t nc,
                      const or_params *p, int32_t *out_ids, float *out_d, or_trace *tr) {
  or_fpair *A = (or_fpair *)malloc(sizeof(or_fpair) * (size_t)(nc > 0 ? nc : 1));
  or_fpair *R = (or_fpair *)malloc(sizeof(or_fpair) * (size_t)(nc > 0 ? nc : 1));
  if (!A || !R) { free(A); free(R); return OR_ENOMEM; }
  /* Stage 2: asymmetric refinement, A <- sort by d^a (Alg2 l.10-13) */
  for (int32_t i = 0; i < nc; ++i) {
    A[i].id = cids[i];
    A[i].v = asym_dist(ix, q, ix->codes + (int64_t)cids[i] * ix->d_pad);
  }
  qsort(A, (size_t)nc, sizeof(or_fpair), cmp_fpair);
  /* Early termination (Alg2 l.15-16; R11) */
  int32_t k = p->k, term = 0;
  if (p->early_term && nc > k) {
    double ak = (double)A[k - 1].v, ak1 = (double)A[k].v;
    double gap = (ak1 - ak) / (ak + 1e-6);
    double ratio = ak1 / (ak + 1e-6);
    term = (gap > p->tau_gap) || (ratio > p->tau_ratio);
  }
  int32_t depth = p->n_rerank < nc ? p->n_rerank : nc;
  /* Adaptive depth ("the system evaluates the spread of asymmetric distances"; reading
   * R27): the ambiguous band around the top-k boundary -- the entries whose d^a lies within a
   * relative tau_spread of d^a_k (fp64 on the fp32 values) -- is re-ranked, never fewer than k */
  if (!isinf(p->tau_spread) && nc > 0) {
    const int32_t kk = k < nc ? k : nc;
    const double thr = (double)A[kk - 1].v * (1.0 + p->tau_spread);
    int32_t band = 0;
    while (band < nc && (double)A[band].v <= thr) ++band;
    if (band < kk) band = kk;
    if (band < depth) depth = band;
  }
  if (term && depth > k) depth = k;  /* "exact reranking is limited to at most k" */
  /* Stage 3: exact distances for the first `depth` entries of A (Alg2 l.19-22) */
  int32_t nr = 0;
  for (int32_t i = 0; i < depth; ++i) {
    R[nr].id = A[i].id;
    R[nr].v = exact_dist(ix, q, ix->base + (int64_t)A[i].id * ix->d);
    if (tr && tr->exact_d) tr->exact_d[i] = R[nr].v;
    ++nr;
  }
  /* Assembly (Alg2 l.23-24): R <- R_exact U remaining from A; top-k of sorted R. */
  if (p->assemble_mode == 0) {
    /* fill reading (R10): A's next entries only "as needed to ensure at least k" */
    for (int32_t i = depth; i < nc && nr < k; ++i) R[nr++] = A[i];
  } else {
    for (int32_t i = depth; i < nc; ++i) R[nr++] = A[i];
  }
  qsort(R, (size_t)nr, sizeof(or_fpair), cmp_fpair);
  for (int32_t i = 0; i < k; ++i) {
    if (i < nr) { out_ids[i] = R[i].id; out_d[i] = R[i].v; }
    else { out_ids[i] = -1; out_d[i] = INFINITY; }
  }
  if (tr) {
    if (tr->asym_ids) for (int32_t i = 0; i < nc; ++i) tr->asym_ids[i] = A[i].id;
    if (tr->asym_d) for (int32_t i = 0; i < nc; ++i) tr->asym_d[i] = A[i].v;
    if (tr->counters) { tr->counters[C_DEPTH] = depth; tr->counters[C_ET] = term; tr->counters[C_NA] = nc; }
  }
  free(A);
  free(R);
  return OR_OK;
}

/* One query through Alg2: quantize (l.4), Stage 1 (l.6-7: greedy upper layers + layer-0
 * beam with ef), C = first min(N_c, |W|) of W, then rerank_one. */
static int search_one(const or_index *ix, const float *q, const or_params *p, uint8_t *qc,
                      uint8_t *visited, or_went *W, int32_t *cids, int32_t *out_ids, float *out_d,
                      or_trace *tr) {
  or_encode(q, 1, ix->d, ix->min_f, ix->scale_f, qc, ix->d_pad);
  int32_t dep;
  int64_t *cnt = tr ? tr->counters : NULL;
  int32_t ep = greedy(ix, qc, &dep, cnt, tr);
  memset(visited, 0, (size_t)ix->n);
  int32_t wsz = (p->beam_form == 1) ? beam_heap(ix, qc, ep, dep, p->ef, visited, W, tr)
                                    : beam_flag(ix, qc, ep, dep, p->ef, visited, W, tr);
  int32_t nc = p->n_coarse < wsz ? p->n_coarse : wsz;
  for (int32_t i = 0; i < nc; ++i) {
    cids[i] = W[i].id;
    if (tr && tr->coarse_ids) tr->coarse_ids[i] = W[i].id;
    if (tr && tr->coarse_dq) tr->coarse_dq[i] = W[i].d;
  }
  if (cnt) cnt[C_NC] = nc;
  return rerank_one(ix, q, cids, nc, p, out_ids, out_d, tr);
}

/* ------------------------------------------------------------------------------------ */
/* FP32-HNSW baseline (the paper's comparison system "HNSW"):   */
/* the same greedy descent and layer-0 beam, on exact fp32 distances, result = the first   */
/* k of W (no quantizer, no re-rank).                                                       */
/* ------------------------------------------------------------------------------------ */

/* Exact fp32 distance in the canonical order R(L) (R22): the padded
 * row (d8 = d rounded up to 8) is cut into 8-float chunks; chunk t belongs to partial l = t mod
 * L; partial l accumulates its chunks in increasing t, elements in increasing j, one FMA per
 * element; then for off = L/2 .. 1 every partial becomes p[l] + p[l ^ off]; the result
 * is p[0].  L = the smallest power of two >= the chunk count, capped at 32.  L2: sum (q - x)^2;
 * inner product: 1 - sum q x (R12). */
static float fp_dist_RL(const float *q, const float *x, int32_t d, int32_t metric) {
  int32_t nch = (d + 7) / 8, L = 1;
  while (L < nch) L *= 2;
  if (L > 32) L = 32;
  float p[32], t2[32];
  for (int32_t l = 0; l < L; ++l) {
    float acc = 0.0f;
    for (int32_t t = l; t < nch; t += L) {
      for (int32_t j = 8 * t; j < 8 * t + 8 && j < d; ++j) {
        if (metric == 0) {
          float e = q[j] - x[j];
          acc = fmaf(e, e, acc);
        } else {
          acc = fmaf(q[j], x[j], acc);
        }
      }
    }
    p[l] = acc;
  }
  for (int32_t off = L / 2; off >= 1; off /= 2) {
    for (int32_t l = 0; l < L; ++l) t2[l] = p[l] + p[l ^ off];
    for (int32_t l = 0; l < L; ++l) p[l] = t2[l];
  }
  return metric == 0 ? p[0] : 1.0f - p[0];
}

static int fkey_less(float da, int32_t ia, float db, int32_t ib) {
  return (da < db) || (da == db && ia < ib);
}

typedef struct { float d; int32_t id; uint8_t expanded; } or_fent;

/* greedy descent + flag-form beam on exact distances (same algorithm as greedy / beam_flag) */
static int search_one_fp(const or_index *ix, const float *q, const or_params *p, uint8_t *visited,
                         or_fent *W, int32_t *out_ids, float *out_d, or_trace *tr) {
  int64_t *cnt = tr ? tr->counters : NULL;
  int32_t cur = ix->entry_point;
  float dcur = fp_dist_RL(q, ix->base + (int64_t)cur * ix->d, ix->d, ix->metric);
  if (cnt) cnt[C_UPPER_EVALS] += 1;
  for (int32_t L = ix->max_level; L >= 1; --L) {
    for (;;) {
      int32_t cap;
      const int32_t *row = nbr_row(ix, cur, L, &cap);
      int32_t best = cur, deg = 0;
      float dbest = dcur;
      for (int32_t t = 0; t < cap; ++t) {
        int32_t u = row[t];
        if (u < 0) continue;
        ++deg;
        float du = fp_dist_RL(q, ix->base + (int64_t)u * ix->d, ix->d, ix->metric);
        if (cnt) cnt[C_UPPER_EVALS] += 1;
        if (fkey_less(du, u, dbest, best)) { best = u; dbest = du; }
      }
      if (cnt) { cnt[C_UPPER_EXP] += 1; cnt[C_UPPER_DEG_SUM] += deg; }
      if (best == cur) break;
      cur = best;
      dcur = dbest;
    }
    if (tr && tr->upper_end && ix->max_level - L < tr->upper_cap) tr->upper_end[ix->max_level - L] = cur;
  }
  memset(visited, 0, (size_t)ix->n);
  int32_t size = 1, ef = p->ef, nexp = 0;
  W[0].d = dcur; W[0].id = cur; W[0].expanded = 0;
  visited[cur] = 1;
  for (;;) {
    int32_t ci = -1;
    for (int32_t i = 0; i < size; ++i)
      if (!W[i].expanded) { ci = i; break; }
    if (ci < 0) break;
    W[ci].expanded = 1;
    int32_t c = W[ci].id;
    if (tr && tr->exp_ids && nexp < tr->exp_cap) tr->exp_ids[nexp] = c;
    ++nexp;
    int32_t cap;
    const int32_t *row = nbr_row(ix, c, 0, &cap);
    int32_t deg = 0;
    for (int32_t t = 0; t < cap; ++t) {
      int32_t u = row[t];
      if (u < 0) continue;
      ++deg;
      if (visited[u]) continue;
      visited[u] = 1;
      float du = fp_dist_RL(q, ix->base + (int64_t)u * ix->d, ix->d, ix->metric);
      if (cnt) cnt[C_EVALS] += 1;
      if (size < ef || fkey_less(du, u, W[size - 1].d, W[size - 1].id)) {
        int32_t pos = size < ef ? size : ef - 1;
        while (pos > 0 && fkey_less(du, u, W[pos - 1].d, W[pos - 1].id)) {
          W[pos] = W[pos - 1];
          --pos;
        }
        W[pos].d = du; W[pos].id = u; W[pos].expanded = 0;
        if (size < ef) ++size;
      }
    }
    if (cnt) cnt[C_DEG_SUM] += deg;
  }
  if (cnt) { cnt[C_EXPANSIONS] += nexp; cnt[C_NC] = size < p->n_coarse ? size : p->n_coarse; }
  int32_t nc = p->n_coarse < size ? p->n_coarse : size;
  for (int32_t i = 0; i < nc; ++i) {
    if (tr && tr->coarse_ids) tr->coarse_ids[i] = W[i].id;
    if (tr && tr->coarse_dq) memcpy(&tr->coarse_dq[i], &W[i].d, sizeof(float));  /* the fp32 bits */
  }
  for (int32_t i = 0; i < p->k; ++i) {
    if (i < size) { out_ids[i] = W[i].id; out_d[i] = W[i].d; }
    else { out_ids[i] = -1; out_d[i] = INFINITY; }
  }
  return OR_OK;
}

float or_dist_fp_RL(const float *q, const float *x, int32_t d, int32_t metric) {
  return fp_dist_RL(q, x, d, metric);
}

static int check_params(const or_params *p) {
  if (p->k < 1 || p->n_coarse < p->k || p->ef < p->n_coarse || p->n_rerank < 0 ||
      p->n_rerank > p->n_coarse || p->tau_gap < 0 || p->tau_ratio < 1 || !(p->tau_spread >= 0))
    return OR_EINVAL;
  return OR_OK;
}

/* Batch entry: nq queries, outputs [nq x k]; optional traces laid out per query
 * (upper_end [nq x upper_cap]: the node where the descent leaves layer L, at max_level - L):
 *   exp_ids [nq x exp_cap], exp_n [nq], coarse_ids/coarse_dq/asym_ids/asym_d/exact_d
 *   [nq x n_coarse], counters [nq x OR_NCOUNT]. */
int or_search(const or_index *ix, const float *q, int64_t nq, const or_params *p,
              int32_t *out_ids, float *out_d, int32_t exp_cap, int32_t *exp_ids,
              int32_t *coarse_ids, int32_t *coarse_dq, int32_t *asym_ids, float *asym_d,
              float *exact_d, int64_t *counters, int32_t upper_cap, int32_t *upper_end) {
  if (check_params(p)) return OR_EINVAL;
  uint8_t *qc = (uint8_t *)calloc((size_t)ix->d_pad, 1);
  uint8_t *visited = (uint8_t *)malloc((size_t)ix->n);
  or_went *W = (or_went *)malloc(sizeof(or_went) * (size_t)(p->ef + 1));
  or_fent *WF = (or_fent *)malloc(sizeof(or_fent) * (size_t)(p->ef + 1));
  int32_t *cids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(p->n_coarse + 1));
  if (!qc || !visited || !W || !WF || !cids) {
    free(qc); free(visited); free(W); free(WF); free(cids);
    return OR_ENOMEM;
  }
  int st = OR_OK;
  for (int64_t i = 0; i < nq && st == OR_OK; ++i) {
    or_trace tr;
    int64_t nc = p->n_coarse;
    tr.exp_cap = exp_cap;
    tr.exp_ids = exp_ids ? exp_ids + i * exp_cap : NULL;
    tr.coarse_ids = coarse_ids ? coarse_ids + i * nc : NULL;
    tr.coarse_dq = coarse_dq ? coarse_dq + i * nc : NULL;
    tr.asym_ids = asym_ids ? asym_ids + i * nc : NULL;
    tr.asym_d = asym_d ? asym_d + i * nc : NULL;
    tr.exact_d = exact_d ? exact_d + i * nc : NULL;
    tr.counters = counters ? counters + i * OR_NCOUNT : NULL;
    tr.upper_cap = upper_cap;
    tr.upper_end = upper_end ? upper_end + i * upper_cap : NULL;
    if (tr.counters) memset(tr.counters, 0, sizeof(int64_t) * OR_NCOUNT);
    if (p->traversal == 1)
      st = search_one_fp(ix, q + i * ix->d, p, visited, WF, out_ids + i * p->k, out_d + i * p->k, &tr);
    else
      st = search_one(ix, q + i * ix->d, p, qc, visited, W, cids, out_ids + i * p->k,
                      out_d + i * p->k, &tr);
  }
  free(qc); free(visited); free(W); free(WF); free(cids);
  return st;
}

/* Standalone Stages 2/ET/3/assembly on caller-supplied C lists ([nq x nc], sorted by
 * (d^q,id), -1 padded; the first -1 ends a list). */
int or_rerank(const or_index *ix, const float *q, int64_t nq, const int32_t *cand, int32_t nc,
              const or_params *p, int32_t *out_ids, float *out_d) {
  if (p->k < 1 || p->n_rerank < 0) return OR_EINVAL;
  int st = OR_OK;
  for (int64_t i = 0; i < nq && st == OR_OK; ++i) {
    const int32_t *c = cand + i * nc;
    int32_t m = 0;
    while (m < nc && c[m] >= 0) ++m;
    st = rerank_one(ix, q + i * ix->d, c, m, p, out_ids + i * p->k, out_d + i * p->k, NULL);
  }
  return st;
}

/* Cross-shard merge (BJ configs[4]): per query, concatenate S lists of k (dist, global id),
 * sort by (dist, id), keep k.  -1 ids (padding) are dropped. */
int or_merge_topk(const float *dist, const int32_t *ids, int32_t n_lists, int64_t nq, int32_t k,
                  float *out_d, int32_t *out_ids) {
  or_fpair *buf = (or_fpair *)malloc(sizeof(or_fpair) * (size_t)n_lists * (size_t)k);
  if (!buf) return OR_ENOMEM;
  for (int64_t i = 0; i < nq; ++i) {
    int32_t m = 0;
    for (int32_t s = 0; s < n_lists; ++s)
      for (int32_t t = 0; t < k; ++t) {
        int64_t o = ((int64_t)s * nq + i) * k + t;
        if (ids[o] < 0) continue;
        buf[m].v = dist[o]; buf[m].id = ids[o]; ++m;
      }
    qsort(buf, (size_t)m, sizeof(or_fpair), cmp_fpair);
    for (int32_t t = 0; t < k; ++t) {
      out_d[i * k + t] = t < m ? buf[t].v : INFINITY;
      out_ids[i * k + t] = t < m ? buf[t].id : -1;
    }
  }
  free(buf);
  return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* brute force references used as pins (tests only)                                      */
/* ------------------------------------------------------------------------------------ */

/* exact top-k by fp64 squared L2 (metric 0) or by 1 - <q,x> (metric 1), ties by id */
int or_bruteforce(const float *x, int64_t n, int32_t d, const float *q, int64_t nq, int32_t k,
                  int32_t metric, int32_t *out_ids, double *out_d) {
  or_dpair *buf = (or_dpair *)malloc(sizeof(or_dpair) * (size_t)n);
  if (!buf) return OR_ENOMEM;
  for (int64_t i = 0; i < nq; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int32_t t = 0; t < d; ++t) {
        if (metric == 0) {
          double e = (double)q[i * d + t] - (double)x[j * d + t];
          acc = acc + e * e;
        } else {
          acc = acc + (double)q[i * d + t] * (double)x[j * d + t];
        }
      }
      buf[j].v = metric == 0 ? acc : 1.0 - acc;
      buf[j].id = j;
    }
    qsort(buf, (size_t)n, sizeof(or_dpair), cmp_dpair);
    for (int32_t t = 0; t < k; ++t) {
      out_ids[i * k + t] = t < n ? (int32_t)buf[t].id : -1;
      out_d[i * k + t] = t < n ? buf[t].v : INFINITY;
    }
  }
  free(buf);
  return OR_OK;
}

/* brute-force top-k by the integer quantized distance (d^q, id) over all codes */
int or_bruteforce_dq(const uint8_t *codes, int64_t n, int32_t d, int32_t d_pad, const uint8_t *qc,
                     int64_t nq, int32_t k, int32_t *out_ids, int32_t *out_d) {
  or_dpair *buf = (or_dpair *)malloc(sizeof(or_dpair) * (size_t)n);
  if (!buf) return OR_ENOMEM;
  for (int64_t i = 0; i < nq; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      buf[j].v = (double)dq_dist(qc + i * d_pad, codes + j * d_pad, d);
      buf[j].id = j;
    }
    qsort(buf, (size_t)n, sizeof(or_dpair), cmp_dpair);
    for (int32_t t = 0; t < k; ++t) {
      out_ids[i * k + t] = t < n ? (int32_t)buf[t].id : -1;
      out_d[i * k + t] = t < n ? (int32_t)buf[t].v : -1;
    }
  }
  free(buf);
  return OR_OK;
}

/* ==================================================================================== */
/* Build phase, Stage 3: graph construction (Alg1 l.16-22) -- the ORACLE of the    */
/* GPU index build.  HNSW insertion [23] over the quantized codes  */
/* with d^q and (d, id) ties, in the wave order of DESIGN.md R28: nodes are inserted in id     */
/* order in batches; every node of a batch searches the graph as it stood when the batch began */
/* and chooses its own neighbours; then the reverse links of the batch are applied per (layer, */
/* target row), sources in id order, pruning a full row with the same selection rule.         */
/* ==================================================================================== */

/* level of a node from its uniform draw u in (0, 1]: floor(-ln(u) / ln(M)), cap 30 */
void or_build_levels(const double *u, int64_t n, int32_t M, int32_t *levels) {
  for (int64_t i = 0; i < n; ++i) {
    double lv = floor(-log(u[i]) * (1.0 / log((double)M)));
    levels[i] = lv > 30.0 ? 30 : (int32_t)lv;
  }
}

typedef struct {
  const uint8_t *codes;
  int64_t n;
  int32_t d, d_pad, M, cap0;
  const int32_t *levels;
  const int64_t *upper_off;
  int32_t *adj0, *adj_upper;
  uint32_t *stamp;   /* visited marks of the current layer search */
  uint32_t epoch;
} or_bgraph;

static int32_t *brow(const or_bgraph *g, int64_t v, int32_t L) {
  return L == 0 ? g->adj0 + v * g->cap0 : g->adj_upper + (g->upper_off[v] + L - 1) * g->M;
}
static int32_t bdist(const or_bgraph *g, int64_t a, int64_t b) {
  return dq_dist(g->codes + a * g->d_pad, g->codes + b * g->d_pad, g->d);
}

/* SEARCH-LAYER [23] in the flag form (R8) from several entry points (sorted by
 * (d, id)): W starts as the ef smallest of them, all unexpanded, and all are marked visited.
 * Rows end at their first -1.  Returns |W|; W sorted by (d, id). */
static int32_t bsearch_layer(or_bgraph *g, int64_t q, const or_went *eps, int32_t n_eps, int32_t ef, int32_t L,
                             or_went *W) {
  if (++g->epoch == 0) { memset(g->stamp, 0, sizeof(uint32_t) * (size_t)g->n); g->epoch = 1; }
  int32_t size = 0;
  for (int32_t i = 0; i < n_eps; ++i) {
    g->stamp[eps[i].id] = g->epoch;
    if (size < ef) { W[size] = eps[i]; W[size].expanded = 0; ++size; }
  }
  const int32_t cap = L == 0 ? g->cap0 : g->M;
  for (;;) {
    int32_t ci = -1;
    for (int32_t i = 0; i < size; ++i)
      if (!W[i].expanded) { ci = i; break; }
    if (ci < 0) break;
    W[ci].expanded = 1;
    const int32_t *row = brow(g, W[ci].id, L);
    for (int32_t t = 0; t < cap; ++t) {
      int32_t u = row[t];
      if (u < 0) break;
      if (g->stamp[u] == g->epoch) continue;
      g->stamp[u] = g->epoch;
      int32_t du = bdist(g, q, u);
      if (size < ef || key_less(du, u, W[size - 1].d, W[size - 1].id)) {
        int32_t pos = size < ef ? size : ef - 1;
        while (pos > 0 && key_less(du, u, W[pos - 1].d, W[pos - 1].id)) { W[pos] = W[pos - 1]; --pos; }
        W[pos].d = du; W[pos].id = u; W[pos].expanded = 0;
        if (size < ef) ++size;
      }
    }
  }
  return size;
}

/* Malkov's neighbour-selection heuristic (R14): scan the candidates in (d, id) order (d = distance
 * to the base node); keep e unless an already kept r is strictly closer to e than the base is
 * (d(e, r) < d(e)); stop at m kept.  keep_pruned: fill the free slots with the rejected ones, in
 * scan order.  Returns the number written to out. */
static int32_t bselect(const or_bgraph *g, const or_went *cand, int32_t nc, int32_t m, int32_t keep_pruned,
                       int32_t *out, int32_t *pruned) {
  int32_t ns = 0, np = 0;
  for (int32_t i = 0; i < nc && ns < m; ++i) {
    int32_t good = 1;
    for (int32_t j = 0; j < ns; ++j)
      if (bdist(g, cand[i].id, out[j]) < cand[i].d) { good = 0; break; }
    if (good) out[ns++] = cand[i].id;
    else if (keep_pruned) pruned[np++] = cand[i].id;
  }
  for (int32_t i = 0; i < np && ns < m; ++i) out[ns++] = pruned[i];
  return ns;
}

typedef struct { int32_t L, target, src; } or_rev;
static int cmp_rev(const void *a, const void *b) {
  const or_rev *x = (const or_rev *)a, *y = (const or_rev *)b;
  if (x->L != y->L) return x->L < y->L ? -1 : 1;
  if (x->target != y->target) return x->target < y->target ? -1 : 1;
  return (x->src > y->src) - (x->src < y->src);
}
static int cmp_went(const void *a, const void *b) {
  const or_went *x = (const or_went *)a, *y = (const or_went *)b;
  if (x->d != y->d) return x->d < y->d ? -1 : 1;
  return (x->id > y->id) - (x->id < y->id);
}

/* Build the graph.  upper_off (out): row of (v, layer 1) in adj_upper, rows of a node consecutive,
 * nodes in id order; adj0 [n x 2M], adj_upper [sum of levels x M] -1 padded (caller-sized, see
 * or_build_upper_rows).  flags bit 0: keep pruned connections; bit 1: a new node selects 2M (not M)
 * layer-0 neighbours.  batch_div: batch = min(max(1, pos / batch_div), 4096) nodes (R28); a node
 * that raises the top level is inserted alone.  entry_max (out) = {entry point, max level}. */
int64_t or_build_upper_rows(const int32_t *levels, int64_t n, int64_t *upper_off) {
  int64_t rows = 0;
  for (int64_t i = 0; i < n; ++i) { upper_off[i] = levels[i] > 0 ? rows : -1; rows += levels[i]; }
  return rows;
}

int or_build_graph(const uint8_t *codes, int64_t n, int32_t d, int32_t d_pad, const int32_t *levels,
                   const int64_t *upper_off, int32_t M, int32_t efc, int32_t flags, int32_t batch_div,
                   int32_t *adj0, int32_t *adj_upper, int32_t *entry_max) {
  if (!codes || n < 1 || M < 2 || efc < 1 || !adj0 || !entry_max) return OR_EINVAL;
  const int32_t keep_pruned = flags & 1, sel0 = (flags & 2) ? 2 * M : M, cap0 = 2 * M;
  if (batch_div <= 0) batch_div = 32;
  int64_t rows = 0;
  for (int64_t i = 0; i < n; ++i) rows += levels[i];
  for (int64_t i = 0; i < n * cap0; ++i) adj0[i] = -1;
  for (int64_t i = 0; i < rows * M; ++i) adj_upper[i] = -1;
  or_bgraph g = {codes, n, d, d_pad, M, cap0, levels, upper_off, adj0, adj_upper, NULL, 0};
  const int32_t wcap = (efc > cap0 ? efc : cap0) + 4096 + 8;
  g.stamp = (uint32_t *)calloc((size_t)n, sizeof(uint32_t));
  or_went *W = (or_went *)malloc(sizeof(or_went) * (size_t)wcap);
  or_went *E = (or_went *)malloc(sizeof(or_went) * (size_t)wcap);
  int32_t *sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)wcap);
  int32_t *pr = (int32_t *)malloc(sizeof(int32_t) * (size_t)wcap);
  or_rev *rev = (or_rev *)malloc(sizeof(or_rev) * (size_t)4096 * (size_t)(31 * M + sel0));
  if (!g.stamp || !W || !E || !sel || !pr || !rev) {
    free(g.stamp); free(W); free(E); free(sel); free(pr); free(rev);
    return OR_ENOMEM;
  }
  int32_t entry = 0, max_level = levels[0];
  int64_t pos = 1;
  while (pos < n) {
    int64_t B = pos / batch_div;
    if (B < 1) B = 1;
    if (B > 4096) B = 4096;
    if (B > n - pos) B = n - pos;
    for (int64_t i = 0; i < B; ++i)
      if (levels[pos + i] > max_level) { B = i == 0 ? 1 : i; break; }
    int64_t nrev = 0;
    /* phase 1: each node of the batch, on the graph as it stood when the batch began (no node of
     * the batch is linked from the graph yet, so the batch cannot see itself) */
    for (int64_t bi = 0; bi < B; ++bi) {
      const int64_t q = pos + bi;
      const int32_t lq = levels[q];
      int32_t cur = entry, dcur = bdist(&g, q, cur);
      for (int32_t L = max_level; L > lq; --L) {  /* greedy descent above the node's level (O9) */
        for (;;) {
          const int32_t *row = brow(&g, cur, L);
          int32_t best = cur, db = dcur;
          for (int32_t t = 0; t < M; ++t) {
            int32_t u = row[t];
            if (u < 0) break;
            int32_t du = bdist(&g, q, u);
            if (key_less(du, u, db, best)) { best = u; db = du; }
          }
          if (best == cur) break;
          cur = best;
          dcur = db;
        }
      }
      int32_t ne = 1;
      E[0].d = dcur; E[0].id = cur; E[0].expanded = 0;
      for (int32_t L = lq < max_level ? lq : max_level; L >= 0; --L) {
        int32_t nw = bsearch_layer(&g, q, E, ne, efc, L, W);
        int32_t m = bselect(&g, W, nw, L == 0 ? sel0 : M, keep_pruned, sel, pr);
        int32_t *row = brow(&g, q, L);
        for (int32_t t = 0; t < m; ++t) {
          row[t] = sel[t];
          rev[nrev].L = L; rev[nrev].target = sel[t]; rev[nrev].src = (int32_t)q; ++nrev;
        }
        memcpy(E, W, sizeof(or_went) * (size_t)nw);  /* the next layer starts from this W */
        ne = nw;
      }
    }
    /* phase 2: reverse links per (layer, target), sources in id order (R28) */
    qsort(rev, (size_t)nrev, sizeof(or_rev), cmp_rev);
    for (int64_t a = 0; a < nrev;) {
      int64_t b = a;
      while (b < nrev && rev[b].L == rev[a].L && rev[b].target == rev[a].target) ++b;
      const int32_t L = rev[a].L, e = rev[a].target, cap = L == 0 ? cap0 : M;
      int32_t *row = brow(&g, e, L);
      int32_t deg = 0;
      while (deg < cap && row[deg] >= 0) ++deg;
      if (deg + (b - a) <= cap) {
        for (int64_t i = a; i < b; ++i) row[deg++] = rev[i].src;
      } else {
        int32_t nc = 0;
        for (int32_t t = 0; t < deg; ++t) { W[nc].d = bdist(&g, e, row[t]); W[nc].id = row[t]; ++nc; }
        for (int64_t i = a; i < b; ++i) { W[nc].d = bdist(&g, e, rev[i].src); W[nc].id = rev[i].src; ++nc; }
        qsort(W, (size_t)nc, sizeof(or_went), cmp_went);
        int32_t m = bselect(&g, W, nc, cap, keep_pruned, sel, pr);
        for (int32_t t = 0; t < cap; ++t) row[t] = t < m ? sel[t] : -1;
      }
      a = b;
    }
    for (int64_t bi = 0; bi < B; ++bi)
      if (levels[pos + bi] > max_level) { max_level = levels[pos + bi]; entry = (int32_t)(pos + bi); }
    pos += B;
  }
  entry_max[0] = entry;
  entry_max[1] = max_level;
  free(g.stamp); free(W); free(E); free(sel); free(pr); free(rev);
  return OR_OK;
}

int or_ncount(void) { return OR_NCOUNT; }

/* ------------------------------------------------------------------------------------ */
/* single-pair hooks for the pin tests (the same static functions the search uses)       */
/* ------------------------------------------------------------------------------------ */
int32_t or_dist_quantized(const uint8_t *qc, const uint8_t *xc, int32_t d) { return dq_dist(qc, xc, d); }

float or_dist_asym(const float *q, const uint8_t *xc, const float *min_f, const float *scale_f, int32_t d,
                   int32_t metric) {
  or_index ix;
  memset(&ix, 0, sizeof(ix));
  ix.d = d; ix.metric = metric; ix.min_f = min_f; ix.scale_f = scale_f;
  return asym_dist(&ix, q, xc);
}

float or_dist_exact(const float *q, const float *x, int32_t d, int32_t metric) {
  or_index ix;
  memset(&ix, 0, sizeof(ix));
  ix.d = d; ix.metric = metric;
  return exact_dist(&ix, q, x);
}

float or_decode(uint8_t c, float scale, float mn) { return decode_elem(c, scale, mn); }
