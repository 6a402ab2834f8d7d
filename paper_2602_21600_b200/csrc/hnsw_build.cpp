// hnsw_build.cpp -- deterministic, multi-threaded host HNSW builder over the quantized codes.
//
// Algorithm 1 Stage 3: G.Insert(q_i, i, M_i, ef^construction) for i = 1..n,
// with the HNSW insertion of [23]: level draw, greedy descent through the layers
// above the node's level, ef^construction beam at each layer <= level, neighbour selection
// by Malkov's diversity heuristic (R14), reverse links with heuristic pruning at
// the degree caps M (layers >= 1) and 2M (layer 0).  Distances are the integer
// quantized distance d^q (Alg2 l.6 without s_dist, R7) with (d, id) tie-breaking.
//
// B200 framing: the graph is an INPUT of the search hot path (north_star: "built once from
// a seed by the host builder, and the same adjacency is fed to both the oracle and the GPU
// path").  It is not on the timed path.  To build 1M-10M nodes on a fresh box in minutes
// the insert loop runs in batches that are deterministic regardless of thread count:
//   phase 1 (parallel over the batch): each new node searches the graph FROZEN at the start
//            of the batch and selects its own neighbours;
//   phase 2 (parallel over target rows): reverse links are grouped by (layer, target) and
//            applied with the heuristic prune; groups are processed in sorted order.
// Batch size grows as pos/32 (capped), and a node that raises the top level is inserted
// alone, so the structure matches sequential insertion up to within-batch visibility.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <thread>
#include <vector>

namespace {

struct Graph {
  int64_t n;
  int32_t d_pad, M, cap0, efc;
  const uint8_t* codes;
  int32_t* levels;
  int64_t* upper_off;
  int32_t* adj0;
  int32_t* adj_upper;
  int32_t entry = -1, max_level = -1;

  inline int32_t dist(int64_t a, int64_t b) const {
    const uint8_t* x = codes + a * d_pad;
    const uint8_t* y = codes + b * d_pad;
    int32_t s = 0;
    for (int32_t j = 0; j < d_pad; ++j) {
      int32_t e = int32_t(x[j]) - int32_t(y[j]);
      s += e * e;
    }
    return s;
  }
  inline int32_t* row(int64_t v, int32_t L) const {
    return L == 0 ? adj0 + v * cap0 : adj_upper + (upper_off[v] + L - 1) * M;
  }
  inline int32_t cap(int32_t L) const { return L == 0 ? cap0 : M; }
};

using Key = std::pair<int32_t, int32_t>;  // (distance, id); lexicographic = (d, id) order

struct Scratch {
  std::vector<uint32_t> stamp;
  uint32_t epoch = 0;
  explicit Scratch(int64_t n) : stamp(size_t(n), 0u) {}
  void next() {
    if (++epoch == 0) { std::fill(stamp.begin(), stamp.end(), 0u); epoch = 1; }
  }
};

// Malkov SEARCH-LAYER (heap form) from a set of entry points; returns W ascending.
std::vector<Key> search_layer(const Graph& g, int64_t q, const std::vector<Key>& eps, int32_t ef,
                              int32_t L, Scratch& s) {
  s.next();
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> C;  // min-heap
  std::priority_queue<Key> W;                                      // max-heap
  for (const Key& e : eps) {
    if (s.stamp[e.second] == s.epoch) continue;
    s.stamp[e.second] = s.epoch;
    C.push(e);
    W.push(e);
    if ((int32_t)W.size() > ef) W.pop();
  }
  while (!C.empty()) {
    Key c = C.top();
    if (c > W.top() && (int32_t)W.size() >= ef) break;
    C.pop();
    const int32_t* r = g.row(c.second, L);
    int32_t cp = g.cap(L);
    for (int32_t t = 0; t < cp; ++t) {
      int32_t u = r[t];
      if (u < 0) break;
      if (s.stamp[u] == s.epoch) continue;
      s.stamp[u] = s.epoch;
      Key ku(g.dist(q, u), u);
      if ((int32_t)W.size() < ef || ku < W.top()) {
        C.push(ku);
        W.push(ku);
        if ((int32_t)W.size() > ef) W.pop();
      }
    }
  }
  std::vector<Key> out;
  out.reserve(W.size());
  while (!W.empty()) { out.push_back(W.top()); W.pop(); }
  std::reverse(out.begin(), out.end());
  return out;
}

// Malkov's neighbour-selection heuristic: scan candidates ascending by distance to the base
// point; keep e unless some already kept r is strictly closer to e than the base is.
// keep_pruned (Malkov's keepPrunedConnections option): fill the remaining slots with the
// closest discarded candidates.
std::vector<int32_t> heuristic(const Graph& g, const std::vector<Key>& cand_sorted, int32_t m, bool keep_pruned) {
  std::vector<int32_t> sel, pruned;
  sel.reserve(m);
  for (const Key& e : cand_sorted) {
    if ((int32_t)sel.size() >= m) break;
    bool good = true;
    for (int32_t r : sel) {
      if (g.dist(e.second, r) < e.first) { good = false; break; }
    }
    if (good) sel.push_back(e.second);
    else if (keep_pruned) pruned.push_back(e.second);
  }
  for (size_t i = 0; i < pruned.size() && (int32_t)sel.size() < m; ++i) sel.push_back(pruned[i]);
  return sel;
}

template <class F>
void parallel_for(int64_t n, int nthreads, F&& fn) {
  if (n <= 0) return;
  if (nthreads <= 1 || n < 4) {
    for (int64_t i = 0; i < n; ++i) fn(i, 0);
    return;
  }
  std::atomic<int64_t> next(0);
  std::vector<std::thread> th;
  int nt = (int)std::min<int64_t>(nthreads, n);
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (;;) {
        int64_t i = next.fetch_add(1);
        if (i >= n) break;
        fn(i, t);
      }
    });
  for (auto& x : th) x.join();
}

struct RevLink {
  int32_t L, target, src;
  bool operator<(const RevLink& o) const {
    if (L != o.L) return L < o.L;
    if (target != o.target) return target < o.target;
    return src < o.src;
  }
};

}  // namespace

#ifndef AQR_SRC_HASH
#define AQR_SRC_HASH "unknown"
#endif

extern "C" {

// the build stamps the hash of this source (build.py: src_hash) so a stale library is rebuilt
const char* aqr_hnsw_version(void) { return "aqr-hnsw-build src:" AQR_SRC_HASH; }

// Level assignment: level_i = floor(-ln(u_i) * mL), mL = 1/ln(M), u_i in (0,1]
// supplied by the caller (seeded); capped at 30.  Fills upper_off (rows of width M for the
// layers 1..level of each node, consecutive) and returns the number of upper rows.
int64_t aqr_hnsw_levels(const double* u, int64_t n, int32_t M, int32_t* levels, int64_t* upper_off) {
  double mL = 1.0 / std::log((double)M);
  int64_t rows = 0;
  for (int64_t i = 0; i < n; ++i) {
    double lv = std::floor(-std::log(u[i]) * mL);
    int32_t l = lv > 30.0 ? 30 : (int32_t)lv;
    levels[i] = l;
    upper_off[i] = l > 0 ? rows : -1;
    rows += l;
  }
  return rows;
}

// Build the graph.  adj0: [n x 2M] and adj_upper: [rows x M] are caller-allocated and are
// filled with -1 padding.  out2 = {entry_point, max_level}.  batch_div: a batch holds at most
// pos / batch_div nodes (0 = 32; a huge value gives sequential insertion).  Returns 0 on success.
int aqr_hnsw_build(const uint8_t* codes, int64_t n, int32_t d_pad, const int32_t* levels,
                   const int64_t* upper_off, int32_t M, int32_t efc, int32_t n_threads,
                   int32_t* adj0, int32_t* adj_upper, int64_t upper_rows, int32_t* out2, int32_t batch_div, int32_t flags) {
  // flags bit 0: keep pruned connections; bit 1: a new node selects 2M (not M) layer-0 neighbours
  const bool keep_pruned = (flags & 1) != 0;
  const int32_t sel0 = (flags & 2) ? 2 * M : M;
  if (!codes || n < 1 || M < 2 || efc < 1 || !adj0 || !out2) return 1;
  Graph g;
  g.n = n; g.d_pad = d_pad; g.M = M; g.cap0 = 2 * M; g.efc = efc; g.codes = codes;
  g.levels = const_cast<int32_t*>(levels);
  g.upper_off = const_cast<int64_t*>(upper_off);
  g.adj0 = adj0;
  g.adj_upper = adj_upper;
  std::fill(adj0, adj0 + n * g.cap0, -1);
  if (adj_upper && upper_rows > 0) std::fill(adj_upper, adj_upper + upper_rows * M, -1);
  if (n_threads <= 0) n_threads = (int)std::max(1u, std::thread::hardware_concurrency());

  std::vector<Scratch> scratch;
  scratch.reserve(n_threads);
  for (int t = 0; t < n_threads; ++t) scratch.emplace_back(n);

  g.entry = 0;
  g.max_level = levels[0];
  int64_t pos = 1;
  const int64_t kBatchCap = 4096;
  if (batch_div <= 0) batch_div = 32;
  std::vector<std::vector<std::pair<int32_t, std::vector<int32_t>>>> sel;  // per batch item: (L, nbrs)
  while (pos < n) {
    int64_t B = std::min<int64_t>(std::max<int64_t>(1, pos / batch_div), kBatchCap);
    B = std::min<int64_t>(B, n - pos);
    for (int64_t i = 0; i < B; ++i)
      if (levels[pos + i] > g.max_level) { B = (i == 0) ? 1 : i; break; }
    sel.assign(size_t(B), {});
    // phase 1: search the frozen graph and choose own neighbours
    parallel_for(B, n_threads, [&](int64_t bi, int tid) {
      int64_t q = pos + bi;
      Scratch& s = scratch[tid];
      int32_t lq = levels[q];
      int32_t cur = g.entry;
      int32_t dcur = g.dist(q, cur);
      for (int32_t L = g.max_level; L > lq; --L) {
        for (;;) {
          const int32_t* r = g.row(cur, L);
          int32_t best = cur, db = dcur;
          for (int32_t t = 0; t < M; ++t) {
            int32_t u = r[t];
            if (u < 0) break;
            int32_t du = g.dist(q, u);
            if (Key(du, u) < Key(db, best)) { best = u; db = du; }
          }
          if (best == cur) break;
          cur = best; dcur = db;
        }
      }
      std::vector<Key> eps{Key(dcur, cur)};
      for (int32_t L = std::min(lq, g.max_level); L >= 0; --L) {
        std::vector<Key> W = search_layer(g, q, eps, efc, L, s);
        std::vector<int32_t> nb = heuristic(g, W, L == 0 ? sel0 : M, keep_pruned);
        int32_t* r = g.row(q, L);
        for (size_t t = 0; t < nb.size(); ++t) r[t] = nb[t];
        sel[bi].emplace_back(L, std::move(nb));
        eps = std::move(W);
      }
    });
    // phase 2: reverse links grouped by (layer, target), applied in sorted order
    std::vector<RevLink> rev;
    for (int64_t bi = 0; bi < B; ++bi)
      for (auto& ln : sel[bi])
        for (int32_t e : ln.second) rev.push_back({ln.first, e, (int32_t)(pos + bi)});
    std::sort(rev.begin(), rev.end());
    std::vector<int64_t> starts;
    for (size_t i = 0; i < rev.size(); ++i)
      if (i == 0 || rev[i].L != rev[i - 1].L || rev[i].target != rev[i - 1].target) starts.push_back((int64_t)i);
    starts.push_back((int64_t)rev.size());
    parallel_for((int64_t)starts.size() - 1, n_threads, [&](int64_t gi, int) {
      int64_t a = starts[gi], b = starts[gi + 1];
      int32_t L = rev[a].L, e = rev[a].target;
      int32_t* r = g.row(e, L);
      int32_t cp = g.cap(L);
      int32_t deg = 0;
      while (deg < cp && r[deg] >= 0) ++deg;
      if (deg + (b - a) <= cp) {
        for (int64_t i = a; i < b; ++i) r[deg++] = rev[i].src;
        return;
      }
      std::vector<Key> cand;
      cand.reserve(size_t(deg + (b - a)));
      for (int32_t t = 0; t < deg; ++t) cand.emplace_back(g.dist(e, r[t]), r[t]);
      for (int64_t i = a; i < b; ++i) cand.emplace_back(g.dist(e, rev[i].src), rev[i].src);
      std::sort(cand.begin(), cand.end());
      std::vector<int32_t> nb = heuristic(g, cand, cp, keep_pruned);
      for (int32_t t = 0; t < cp; ++t) r[t] = t < (int32_t)nb.size() ? nb[t] : -1;
    });
    for (int64_t bi = 0; bi < B; ++bi)
      if (levels[pos + bi] > g.max_level) { g.max_level = levels[pos + bi]; g.entry = (int32_t)(pos + bi); }
    pos += B;
  }
  out2[0] = g.entry;
  out2[1] = g.max_level;
  return 0;
}

}  // extern "C"
