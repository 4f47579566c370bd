// instances.cpp — seeded synthetic-instance generators (host side).
//
// These produce the BASELINE.json workloads deterministically
// from the reference's RNG contract (proj/include/gw/rng.hpp:13-53:
// std::mt19937_64, uniform01 = (x >> 11)·2^-53, unbiased `below`, Box-Muller
// normal with a cached spare).  Generators that exist in the reference follow
// its algorithm exactly (checked edge-for-edge against the reference TUs in
// tests/test_instances.py); the others are new and documented in DESIGN.md.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <numeric>
#include <random>
#include <unordered_set>
#include <utility>
#include <vector>

#include "gwbinst.h"

namespace {

class Rng {  // same draw sequence as gw::Rng (rng.hpp:13-53)
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * uniform01(); }
  uint64_t below(uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t r;
    do {
      r = eng_();
    } while (r >= limit);
    return r % n;
  }
  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1;
    do {
      u1 = uniform01();
    } while (u1 <= 0.0);
    const double u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    spare_ = r * std::sin(2.0 * std::numbers::pi * u2);
    has_spare_ = true;
    return r * std::cos(2.0 * std::numbers::pi * u2);
  }

 private:
  std::mt19937_64 eng_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

using Edge = std::pair<int32_t, int32_t>;

// gw::Graph canonical form (types.cpp:155-174): (min,max), sorted, unique.
void canonicalize(std::vector<Edge>& e) {
  for (auto& [a, b] : e)
    if (a > b) std::swap(a, b);
  std::sort(e.begin(), e.end());
  e.erase(std::unique(e.begin(), e.end()), e.end());
}

int64_t emit(const std::vector<Edge>& e, int32_t* out, int64_t cap) {
  const int64_t n = static_cast<int64_t>(e.size());
  for (int64_t k = 0; k < n && k < cap; ++k) {
    out[2 * k] = e[static_cast<size_t>(k)].first;
    out[2 * k + 1] = e[static_cast<size_t>(k)].second;
  }
  return n;
}

std::vector<Edge> read(const int32_t* edges, int64_t count) {
  std::vector<Edge> e(static_cast<size_t>(count));
  for (int64_t k = 0; k < count; ++k) e[static_cast<size_t>(k)] = {edges[2 * k], edges[2 * k + 1]};
  return e;
}

uint64_t key(int32_t a, int32_t b) {
  if (a > b) std::swap(a, b);
  return (static_cast<uint64_t>(a) << 32) | static_cast<uint32_t>(b);
}

}  // namespace

extern "C" {

// Barabási–Albert graph, algorithm of gen_barabasi_albert (tasks.cpp:22-65).
GWBINST_API int64_t gwbinst_gen_barabasi_albert(int32_t n, int32_t m_attach, uint64_t seed,
                                int32_t* out, int64_t cap) {
  if (m_attach < 1 || m_attach >= n) return -1;
  Rng rng(seed);
  std::vector<Edge> edges;
  std::vector<double> degree(static_cast<size_t>(n), 0.0);
  for (int a = 0; a <= m_attach; ++a)
    for (int b = a + 1; b <= m_attach; ++b) {
      edges.emplace_back(a, b);
      degree[a] += 1.0;
      degree[b] += 1.0;
    }
  std::vector<double> weight(static_cast<size_t>(n), 0.0);
  for (int v = m_attach + 1; v < n; ++v) {
    std::copy(degree.begin(), degree.begin() + v, weight.begin());
    double total = std::accumulate(weight.begin(), weight.begin() + v, 0.0);
    for (int pick = 0; pick < m_attach; ++pick) {
      double r = rng.uniform01() * total;
      int chosen = 0;
      for (int u = 0; u < v; ++u) {
        r -= weight[u];
        chosen = u;
        if (r < 0.0) break;
      }
      edges.emplace_back(chosen, v);
      total -= weight[chosen];
      weight[chosen] = 0.0;
    }
    for (size_t k = edges.size() - m_attach; k < edges.size(); ++k) {
      degree[edges[k].first] += 1.0;
      degree[edges[k].second] += 1.0;
    }
  }
  canonicalize(edges);
  return emit(edges, out, cap);
}

// Erdős–Rényi G(n, p): gen_gaussian_partition(n, 1, p, 0, seed)
// (tasks.cpp:67-112) with a single cluster, which draws the cluster size
// from one Box-Muller normal and then one uniform per pair i<j.
GWBINST_API int64_t gwbinst_gen_erdos_renyi(int32_t n, double p, uint64_t seed, int32_t* out,
                            int64_t cap) {
  Rng rng(seed);
  (void)rng.normal();  // the k=1 cluster-size draw; size is then forced to n
  std::vector<Edge> edges;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (rng.uniform01() < p) edges.emplace_back(i, j);
  return emit(edges, out, cap);
}

// Stochastic block model with k equal blocks (label = i·k/n): new generator
// (the reference's planted partition uses Gaussian block sizes).
GWBINST_API int64_t gwbinst_gen_sbm_equal(int32_t n, int32_t k, double p_in, double p_out,
                          uint64_t seed, int32_t* out, int64_t cap,
                          int32_t* labels) {
  Rng rng(seed);
  std::vector<int32_t> lab(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) lab[i] = static_cast<int32_t>((int64_t)i * k / n);
  if (labels) std::memcpy(labels, lab.data(), sizeof(int32_t) * n);
  std::vector<Edge> edges;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (rng.uniform01() < (lab[i] == lab[j] ? p_in : p_out)) edges.emplace_back(i, j);
  return emit(edges, out, cap);
}

// Edge noise: remove floor(q_remove·|E|) edges (partial Fisher-Yates, as
// add_noise samples, tasks.cpp:131-137) and add floor(q_add·|E|) pairs absent
// from the input graph by rejection sampling (the reference enumerates all
// absent pairs, O(n²) memory, impractical at n = 20000).  New generator.
GWBINST_API int64_t gwbinst_edge_noise(int32_t n, const int32_t* edges, int64_t count,
                       double q_remove, double q_add, uint64_t seed,
                       int32_t* out, int64_t cap) {
  Rng rng(seed);
  std::vector<Edge> e = read(edges, count);
  canonicalize(e);
  const int64_t ne = static_cast<int64_t>(e.size());
  const int64_t n_rem = static_cast<int64_t>(std::floor(q_remove * ne));
  const int64_t n_add = static_cast<int64_t>(std::floor(q_add * ne));
  std::unordered_set<uint64_t> present;
  present.reserve(static_cast<size_t>(2 * ne + n_add + 16));
  for (auto [a, b] : e) present.insert(key(a, b));
  for (int64_t t = 0; t < n_rem; ++t) {
    const uint64_t pick = t + rng.below(static_cast<uint64_t>(ne - t));
    std::swap(e[static_cast<size_t>(t)], e[static_cast<size_t>(pick)]);
  }
  std::vector<Edge> kept(e.begin() + n_rem, e.end());
  const int64_t max_pairs = (int64_t)n * (n - 1) / 2;
  int64_t added = 0;
  while (added < n_add && ne + added < max_pairs) {
    const int32_t a = static_cast<int32_t>(rng.below(static_cast<uint64_t>(n)));
    const int32_t b = static_cast<int32_t>(rng.below(static_cast<uint64_t>(n)));
    if (a == b) continue;
    if (!present.insert(key(a, b)).second) continue;
    kept.emplace_back(std::min(a, b), std::max(a, b));
    ++added;
  }
  canonicalize(kept);
  return emit(kept, out, cap);
}

// Uniform relabeling, algorithm of permute_graph (tasks.cpp:141-154);
// perm maps old index -> new.
GWBINST_API int64_t gwbinst_permute_graph(int32_t n, const int32_t* edges, int64_t count,
                          uint64_t seed, int32_t* out, int32_t* perm) {
  Rng rng(seed);
  std::vector<int32_t> p(static_cast<size_t>(n));
  std::iota(p.begin(), p.end(), 0);
  for (int i = n - 1; i > 0; --i)
    std::swap(p[i], p[rng.below(static_cast<uint64_t>(i) + 1)]);
  std::vector<Edge> e;
  e.reserve(static_cast<size_t>(count));
  for (int64_t k = 0; k < count; ++k) e.emplace_back(p[edges[2 * k]], p[edges[2 * k + 1]]);
  canonicalize(e);
  if (perm) std::memcpy(perm, p.data(), sizeof(int32_t) * n);
  return emit(e, out, count);
}

// 3-D isotropic Gaussian mixture (new generator for config 2): k means
// uniform in [0,1]^3, each point picks a component with `below(k)` and adds
// sigma·N(0, I).  Points are row-major n×3.
GWBINST_API void gwbinst_gen_gmm3d(int32_t n, int32_t k, double sigma, uint64_t seed,
                   double* xyz) {
  Rng rng(seed);
  std::vector<double> means(static_cast<size_t>(3 * k));
  for (auto& v : means) v = rng.uniform01();
  for (int i = 0; i < n; ++i) {
    const uint64_t c = rng.below(static_cast<uint64_t>(k));
    for (int d = 0; d < 3; ++d) xyz[3 * i + d] = means[3 * c + d] + sigma * rng.normal();
  }
}

// Euclidean distance matrix (fp64 math), divided by its max and rounded to
// fp32 so that fp32 and fp64 consumers see identical values.  out: n×n fp32.
GWBINST_API void gwbinst_distance_maxnorm_f32(int32_t n, const double* xyz, float* out) {
  std::vector<double> d(static_cast<size_t>(n) * n);
  double mx = 0.0;
  for (int i = 0; i < n; ++i) {
    d[(size_t)i * n + i] = 0.0;
    for (int j = i + 1; j < n; ++j) {
      const double dx = xyz[3 * i] - xyz[3 * j], dy = xyz[3 * i + 1] - xyz[3 * j + 1],
                   dz = xyz[3 * i + 2] - xyz[3 * j + 2];
      const double v = std::sqrt(dx * dx + dy * dy + dz * dz);
      d[(size_t)i * n + j] = d[(size_t)j * n + i] = v;
      mx = std::max(mx, v);
    }
  }
  for (size_t k = 0; k < d.size(); ++k) out[k] = static_cast<float>(mx > 0 ? d[k] / mx : 0.0);
}

// jittered_product (experiment.cpp:41-58): the reference's seeded start for
// the experiment harness.  Entries are drawn column by column; the sum is a
// plain running sum in the same order.
GWBINST_API void gwbinst_jittered_product(const double* mu, int64_t n, const double* nu, int64_t m,
                                          double jitter, uint64_t seed, double* out) {
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < n; ++i) out[j * n + i] = mu[i] * nu[j];
  if (jitter > 0.0) {
    Rng rng(seed);
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < n; ++i) out[j * n + i] *= 1.0 + jitter * rng.uniform(-1.0, 1.0);
    double total = 0.0;
    for (int64_t k = 0; k < n * m; ++k) total += out[k];
    for (int64_t k = 0; k < n * m; ++k) out[k] /= total;
  }
}

}  // extern "C"
