// graphgen.cpp — seeded synthetic graph generators (shared INPUT generators).
//
// This module holds none of the walk-Laplacian arithmetic: it only produces
// simple, symmetric, unweighted graphs in CSR form (§2, P:74-90:
// "we will only consider simple unweighted graphs"), shaped like the paper's
// networks (Table 1: power-law ca-*/human_gene*, road networks).
// Both the CUDA path (bench, tests) and the CPU oracle (tests) consume the
// exact same bytes produced here.
//
// Determinism: every random draw is a pure function of (seed, stream, index)
// through a counter-based splitmix64 hash, and every parallel step either
// writes disjoint outputs or is followed by a sort on unique keys, so the
// output is bit-identical for any OpenMP thread count.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <parallel/algorithm>
#include <stdexcept>
#include <string>
#include <vector>
#include <omp.h>
#include <chrono>
#include <cstdio>

namespace {

thread_local std::string g_err;
static double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static void vlog(const char* what, double t0) { if (std::getenv("GG_VERBOSE")) std::fprintf(stderr, "[graphgen] %s %.3fs\n", what, now_s() - t0); }

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// counter-based draw: (seed, stream, index) -> 64 random bits
inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t idx) {
  return mix64(mix64(seed ^ mix64(stream)) + idx);
}
inline double u53(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

struct Graph {
  int64_t n = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col_idx;
};

// Build a simple symmetric CSR from canonical unique edges (u < v), sorted.
// Rows are sorted ascending; both directions are stored (row_ptr[n] = 2m).
Graph csr_from_canonical(int64_t n, const std::vector<uint64_t>& keys, int64_t kn) {
  // key = u * kn + v, u < v
  Graph g;
  g.n = n;
  const int64_t m = (int64_t)keys.size();
  std::vector<int64_t> deg(n + 1, 0);
  {
    std::vector<std::atomic<int64_t>> d(n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) d[i].store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
      int64_t u = (int64_t)(keys[e] / (uint64_t)kn), v = (int64_t)(keys[e] % (uint64_t)kn);
      d[u].fetch_add(1, std::memory_order_relaxed);
      d[v].fetch_add(1, std::memory_order_relaxed);
    }
    for (int64_t i = 0; i < n; ++i) deg[i] = d[i].load();
  }
  g.row_ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) g.row_ptr[i + 1] = g.row_ptr[i] + deg[i];
  g.col_idx.assign((size_t)g.row_ptr[n], 0);
  {
    std::vector<std::atomic<int64_t>> pos(n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) pos[i].store(g.row_ptr[i], std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
      int64_t u = (int64_t)(keys[e] / (uint64_t)kn), v = (int64_t)(keys[e] % (uint64_t)kn);
      g.col_idx[pos[u].fetch_add(1, std::memory_order_relaxed)] = (int32_t)v;
      g.col_idx[pos[v].fetch_add(1, std::memory_order_relaxed)] = (int32_t)u;
    }
  }
  // per-row sort makes the (thread-order dependent) fill deterministic
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    std::sort(g.col_idx.begin() + g.row_ptr[i], g.col_idx.begin() + g.row_ptr[i + 1]);
  return g;
}

void sort_unique(std::vector<uint64_t>& k) {
  __gnu_parallel::sort(k.begin(), k.end());
  k.erase(std::unique(k.begin(), k.end()), k.end());
}

// ---------------------------------------------------------------------------
// R-MAT (Chakrabarti et al.): recursive quadrant choice with probabilities
// (a, b, c, d = 1-a-b-c) over 2^scale ids; ids >= n rejected, loops dropped,
// undirected duplicates merged.  Candidate edges are generated in index
// batches of size m until at least m unique edges exist; exactly m are then
// kept (the m smallest hash(key) values — a seeded uniform subset).  Finally
// ids are relabelled by a seeded random permutation (perm_seed; 0 = none).
Graph rmat(int scale, int64_t n, int64_t m, double a, double b, double c, uint64_t seed,
           uint64_t perm_seed) {
  if (scale < 1 || scale > 31 || n < 2 || n > (int64_t(1) << scale) || m < 1)
    throw std::runtime_error("rmat: bad size arguments");
  if (m > n * (n - 1) / 2) throw std::runtime_error("rmat: m exceeds n(n-1)/2");
  if (n > INT32_MAX) throw std::runtime_error("rmat: n must fit int32 column ids");
  const double ab = a + b, abc = a + b + c;
  std::vector<uint64_t> uniq;
  const uint64_t kn = (uint64_t)n;
  double t0 = now_s();
  for (uint64_t batch = 0;; ++batch) {
    if (batch > 64) throw std::runtime_error("rmat: could not reach m unique edges");
    std::vector<uint64_t> cand((size_t)m);
    const uint64_t base = batch * (uint64_t)m;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
      const uint64_t idx = base + (uint64_t)e;
      uint64_t u = 0, v = 0;
      for (int l = 0; l < scale; l += 2) {
        uint64_t x = draw(seed, 0x52'4D'41'54ull /*"RMAT"*/, idx * 16 + (uint64_t)(l >> 1));
        for (int h = 0; h < 2 && l + h < scale; ++h) {
          const double r = (double)(h == 0 ? (x >> 32) : (x & 0xffffffffull)) * 0x1.0p-32;
          // quadrant: [0,a) -> (0,0), [a,a+b) -> (0,1), [a+b,a+b+c) -> (1,0), else (1,1)
          const uint64_t bu = (uint64_t)(r >= ab);
          const uint64_t bv = (uint64_t)((r >= a) & (r < ab)) | (uint64_t)(r >= abc);
          u = (u << 1) | bu;
          v = (v << 1) | bv;
        }
      }
      if (u >= kn || v >= kn || u == v) { cand[e] = UINT64_MAX; continue; }
      if (u > v) std::swap(u, v);
      cand[e] = u * kn + v;
    }
    vlog("rmat batch draws", t0);
    sort_unique(cand);
    const size_t mid = uniq.size();
    uniq.insert(uniq.end(), cand.begin(), cand.end());
    std::vector<uint64_t>().swap(cand);
    std::inplace_merge(uniq.begin(), uniq.begin() + (ptrdiff_t)mid, uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    vlog("rmat batch sort_unique", t0);
    if (!uniq.empty() && uniq.back() == UINT64_MAX) uniq.pop_back();
    if ((int64_t)uniq.size() >= m) break;
  }
  if ((int64_t)uniq.size() > m) {
    // seeded uniform subset of exactly m edges: keep the m smallest (hash, key)
    std::vector<std::pair<uint64_t, uint64_t>> hk(uniq.size());
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)uniq.size(); ++i)
      hk[i] = {draw(seed, 0x5355'4253ull /*"SUBS"*/, uniq[i]), uniq[i]};
    __gnu_parallel::nth_element(hk.begin(), hk.begin() + m, hk.end());
    uniq.resize((size_t)m);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) uniq[i] = hk[i].second;
    std::vector<std::pair<uint64_t, uint64_t>>().swap(hk);
    __gnu_parallel::sort(uniq.begin(), uniq.end());
  }
  vlog("rmat subset", t0);
  if (perm_seed != 0) {
    std::vector<std::pair<uint64_t, int64_t>> hp((size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) hp[i] = {draw(perm_seed, 0x5045'524Dull /*"PERM"*/, (uint64_t)i), i};
    __gnu_parallel::sort(hp.begin(), hp.end());
    std::vector<int64_t> newid((size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) newid[hp[k].second] = k;
    std::vector<std::pair<uint64_t, int64_t>>().swap(hp);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
      uint64_t u = (uint64_t)newid[uniq[e] / kn], v = (uint64_t)newid[uniq[e] % kn];
      if (u > v) std::swap(u, v);
      uniq[e] = u * kn + v;
    }
    __gnu_parallel::sort(uniq.begin(), uniq.end());
  }
  vlog("rmat permute", t0);
  Graph g = csr_from_canonical(n, uniq, (int64_t)kn);
  vlog("rmat csr", t0);
  return g;
}

// ---------------------------------------------------------------------------
// Barabasi-Albert preferential attachment: initial star on m0+1 nodes (hub 0),
// then node s = m0+1..n-1 attaches to m0 distinct targets drawn uniformly from
// the degree-weighted multiset ("repeated nodes") of the current graph.
Graph ba(int64_t n, int m0, uint64_t seed) {
  if (m0 < 1 || n < m0 + 2) throw std::runtime_error("ba: need m0 >= 1 and n >= m0+2");
  if (n > INT32_MAX) throw std::runtime_error("ba: n too large");
  std::vector<uint64_t> keys;
  std::vector<int64_t> rep;
  rep.reserve((size_t)(2 * m0 * n));
  for (int64_t j = 1; j <= m0; ++j) {
    keys.push_back(0 * (uint64_t)n + (uint64_t)j);
    rep.push_back(0);
    rep.push_back(j);
  }
  std::vector<int64_t> tg;
  for (int64_t s = m0 + 1; s < n; ++s) {
    tg.clear();
    uint64_t attempt = 0;
    while ((int)tg.size() < m0) {
      uint64_t x = draw(seed, 0x4241ull /*"BA"*/, (uint64_t)s * 4096 + attempt++);
      int64_t t = rep[(size_t)(u53(x) * (double)rep.size())];
      if (std::find(tg.begin(), tg.end(), t) == tg.end()) tg.push_back(t);
      if (attempt > 4000) throw std::runtime_error("ba: target sampling did not terminate");
    }
    for (int64_t t : tg) {
      keys.push_back((uint64_t)t * (uint64_t)n + (uint64_t)s);  // t < s
      rep.push_back(t);
      rep.push_back(s);
    }
  }
  sort_unique(keys);
  return csr_from_canonical(n, keys, n);
}

// ---------------------------------------------------------------------------
// Road-like proxy: nx-by-ny grid (node (i,j) -> i*ny + j), each grid edge
// deleted independently with probability p_del, then the largest connected
// component is kept (ties: the component holding the smallest id) and
// relabelled in increasing original id order.
struct DSU {
  std::vector<int64_t> p;
  explicit DSU(int64_t n) : p((size_t)n) { std::iota(p.begin(), p.end(), 0); }
  int64_t f(int64_t x) {
    while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
    return x;
  }
  void u(int64_t a, int64_t b) {
    a = f(a); b = f(b);
    if (a == b) return;
    if (a < b) std::swap(a, b);
    p[a] = b;  // root = smaller id (deterministic)
  }
};

Graph grid_lcc(int64_t nx, int64_t ny, double p_del, uint64_t seed) {
  if (nx < 1 || ny < 1 || nx * ny < 2) throw std::runtime_error("grid: bad size");
  if (!(p_del >= 0.0 && p_del < 1.0)) throw std::runtime_error("grid: p_del must be in [0,1)");
  const int64_t n = nx * ny;
  std::vector<uint64_t> keys;
  keys.reserve((size_t)(2 * n));
  // horizontal edges (i,j)-(i,j+1) get edge ids [0, nx*(ny-1)); vertical after
  int64_t eid = 0;
  for (int64_t i = 0; i < nx; ++i)
    for (int64_t j = 0; j + 1 < ny; ++j, ++eid)
      if (u53(draw(seed, 0x47524944ull /*"GRID"*/, (uint64_t)eid)) >= p_del)
        keys.push_back((uint64_t)(i * ny + j) * (uint64_t)n + (uint64_t)(i * ny + j + 1));
  for (int64_t i = 0; i + 1 < nx; ++i)
    for (int64_t j = 0; j < ny; ++j, ++eid)
      if (u53(draw(seed, 0x47524944ull, (uint64_t)eid)) >= p_del)
        keys.push_back((uint64_t)(i * ny + j) * (uint64_t)n + (uint64_t)((i + 1) * ny + j));
  DSU d(n);
  for (uint64_t k : keys) d.u((int64_t)(k / (uint64_t)n), (int64_t)(k % (uint64_t)n));
  std::vector<int64_t> csize((size_t)n, 0);
  for (int64_t i = 0; i < n; ++i) csize[d.f(i)]++;
  int64_t best = 0;
  for (int64_t r = 0; r < n; ++r)
    if (csize[r] > csize[best]) best = r;  // strict: smallest root id wins ties
  std::vector<int64_t> nid((size_t)n, -1);
  int64_t nn = 0;
  for (int64_t i = 0; i < n; ++i)
    if (d.f(i) == best) nid[i] = nn++;
  std::vector<uint64_t> k2;
  k2.reserve(keys.size());
  for (uint64_t k : keys) {
    int64_t u = (int64_t)(k / (uint64_t)n), v = (int64_t)(k % (uint64_t)n);
    if (nid[u] >= 0 && nid[v] >= 0) k2.push_back((uint64_t)nid[u] * (uint64_t)nn + (uint64_t)nid[v]);
  }
  sort_unique(k2);
  return csr_from_canonical(nn, k2, nn);
}

// Generic: simplify an arbitrary edge list (drop loops, symmetrize, merge dups).
Graph from_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v) {
  if (n < 1 || n > INT32_MAX) throw std::runtime_error("from_edges: bad n");
  std::vector<uint64_t> keys;
  keys.reserve((size_t)m);
  for (int64_t e = 0; e < m; ++e) {
    int64_t a = u[e], b = v[e];
    if (a < 0 || b < 0 || a >= n || b >= n) throw std::runtime_error("from_edges: id out of range");
    if (a == b) continue;
    if (a > b) std::swap(a, b);
    keys.push_back((uint64_t)a * (uint64_t)n + (uint64_t)b);
  }
  sort_unique(keys);
  return csr_from_canonical(n, keys, n);
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}

}  // namespace

extern "C" {
struct gg_graph { Graph g; };

const char* gg_last_error(void) { return g_err.c_str(); }

int gg_rmat(int scale, int64_t n, int64_t m, double a, double b, double c, uint64_t seed,
            uint64_t perm_seed, gg_graph** out) {
  return guard([&] { *out = new gg_graph{rmat(scale, n, m, a, b, c, seed, perm_seed)}; });
}
int gg_ba(int64_t n, int m0, uint64_t seed, gg_graph** out) {
  return guard([&] { *out = new gg_graph{ba(n, m0, seed)}; });
}
int gg_grid_lcc(int64_t nx, int64_t ny, double p_del, uint64_t seed, gg_graph** out) {
  return guard([&] { *out = new gg_graph{grid_lcc(nx, ny, p_del, seed)}; });
}
int gg_from_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v, gg_graph** out) {
  return guard([&] { *out = new gg_graph{from_edges(n, m, u, v)}; });
}
int64_t gg_n(const gg_graph* h) { return h->g.n; }
int64_t gg_nnz(const gg_graph* h) { return h->g.row_ptr.empty() ? 0 : h->g.row_ptr.back(); }
void gg_copy(const gg_graph* h, int64_t* row_ptr, int32_t* col_idx) {
  std::memcpy(row_ptr, h->g.row_ptr.data(), sizeof(int64_t) * (size_t)(h->g.n + 1));
  std::memcpy(col_idx, h->g.col_idx.data(), sizeof(int32_t) * h->g.col_idx.size());
}
void gg_destroy(gg_graph* h) { delete h; }
void gg_set_threads(int t) { if (t > 0) omp_set_num_threads(t); }
}
