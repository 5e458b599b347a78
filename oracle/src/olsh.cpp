// ORACLE — test infrastructure only. Neighbor graph, particle reorder, LSH
// neighbor search and SVGD restated from /root/reference/proj:
// include/steinmcl/neighbor_graph.hpp:24-90, src/particle_set.cpp:7-47,
// src/neighbor_search.cpp:25-192, src/reference.cpp:78-215, src/svgd.cpp:7-62.
#include <algorithm>
#include <bit>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "oracle.hpp"

namespace orc {

// ---------------------------------------------------------------- graph
void NeighborGraph::init_self(std::size_t n, int k) {  // neighbor_graph.hpp:24-33
  k_max = k;
  idx.assign(n * static_cast<std::size_t>(k), -1);
  kval.assign(n * static_cast<std::size_t>(k), 0.0f);
  count.assign(n, 1);
  for (std::size_t i = 0; i < n; ++i) {
    idx[i * static_cast<std::size_t>(k)] = static_cast<std::int32_t>(i);
    kval[i * static_cast<std::size_t>(k)] = 1.0f;
  }
}

void NeighborGraph::offer(std::size_t i, std::int32_t j, float k_ij) {  // neighbor_graph.hpp:47-73
  const std::size_t base = i * static_cast<std::size_t>(k_max);
  const int n = count[i];
  for (int s = 0; s < n; ++s)
    if (idx[base + static_cast<std::size_t>(s)] == j) return;
  if (n < k_max) {
    idx[base + static_cast<std::size_t>(n)] = j;
    kval[base + static_cast<std::size_t>(n)] = k_ij;
    count[i] = n + 1;
    return;
  }
  const std::int32_t self = static_cast<std::int32_t>(i);
  int weakest = -1;
  float weakest_k = std::numeric_limits<float>::infinity();
  for (int s = 0; s < n; ++s) {
    if (idx[base + static_cast<std::size_t>(s)] == self) continue;
    if (kval[base + static_cast<std::size_t>(s)] < weakest_k) {
      weakest_k = kval[base + static_cast<std::size_t>(s)];
      weakest = s;
    }
  }
  if (weakest >= 0 && k_ij > weakest_k) {
    idx[base + static_cast<std::size_t>(weakest)] = j;
    kval[base + static_cast<std::size_t>(weakest)] = k_ij;
  }
}

void NeighborGraph::refresh(std::size_t i, std::span<const Pose> poses, const KernelParams& kp) {  // 76-90
  const std::size_t base = i * static_cast<std::size_t>(k_max);
  const Pose inv_i = inverse(poses[i]);
  for (int s = 0; s < count[i]; ++s) {
    const std::int32_t j = idx[base + static_cast<std::size_t>(s)];
    float k = 0.0f;
    if (j == static_cast<std::int32_t>(i)) {
      k = 1.0f;
    } else if (!kernel_underflows(poses[i], poses[static_cast<std::size_t>(j)], kp)) {
      k = static_cast<float>(kernel_of_tangent(se3_log(compose(inv_i, poses[static_cast<std::size_t>(j)])), kp));
    }
    kval[base + static_cast<std::size_t>(s)] = k;
  }
}

// particle_set.cpp:7-47
void ParticleSet::reorder(std::span<const std::int32_t> old_of_new) {
  const std::size_t n = size();
  if (old_of_new.size() != n) throw std::invalid_argument("ParticleSet::reorder: permutation size mismatch");
  std::vector<std::int32_t> new_of_old(n);
  for (std::size_t p = 0; p < n; ++p) new_of_old[static_cast<std::size_t>(old_of_new[p])] = static_cast<std::int32_t>(p);
  std::vector<Pose> poses2(n);
  std::vector<double> post2(n);
  std::vector<std::int32_t> id2(n);
  const std::size_t k = static_cast<std::size_t>(neighbors.k_max);
  std::vector<std::int32_t> idx2(n * k);
  std::vector<float> kval2(n * k);
  std::vector<std::int32_t> count2(n);
#pragma omp parallel for schedule(static)
  for (std::int64_t p = 0; p < static_cast<std::int64_t>(n); ++p) {
    const std::size_t dst = static_cast<std::size_t>(p);
    const std::size_t src = static_cast<std::size_t>(old_of_new[dst]);
    poses2[dst] = poses[src];
    post2[dst] = log_post[src];
    id2[dst] = id[src];
    count2[dst] = neighbors.count[src];
    for (int s = 0; s < neighbors.count[src]; ++s) {
      idx2[dst * k + static_cast<std::size_t>(s)] =
          new_of_old[static_cast<std::size_t>(neighbors.idx[src * k + static_cast<std::size_t>(s)])];
      kval2[dst * k + static_cast<std::size_t>(s)] = neighbors.kval[src * k + static_cast<std::size_t>(s)];
    }
  }
  poses.swap(poses2);
  log_post.swap(post2);
  id.swap(id2);
  neighbors.idx.swap(idx2);
  neighbors.kval.swap(kval2);
  neighbors.count.swap(count2);
}

// ---------------------------------------------------------------- LSH
namespace {
constexpr std::uint64_t k_hash_primes[6] = {73856093ull, 19349663ull, 83492791ull,
                                            49979687ull, 39916801ull, 15485863ull};  // neighbor_search.cpp:20-21
}

// neighbor_search.cpp:25-35
std::uint64_t lsh_hash(const Pose& pose, const Pose& frame, const V6& noise, const LshConfig& cfg,
                       const KernelParams& kp) {
  const V6 d = se3_log(compose(inverse(frame), pose));
  const double w[6] = {kp.sigma_r, kp.sigma_r, kp.sigma_r, kp.sigma_t, kp.sigma_t, kp.sigma_t};
  std::uint64_t h = 0;
  for (int c = 0; c < 6; ++c) {
    const double zeta = cfg.alpha * (w[c] * d[c]) + noise[c];
    const double f = std::floor(zeta);
    // static_cast<int64_t> of an out-of-range double is x86 0x8000000000000000.
    const std::int64_t cell = (f >= -9223372036854775808.0 && f < 9223372036854775808.0)
                                  ? static_cast<std::int64_t>(f)
                                  : INT64_MIN;
    h ^= static_cast<std::uint64_t>(cell) * k_hash_primes[c];
  }
  return h;
}

// neighbor_search.cpp:37-44
Pose random_lsh_frame(SplitMix64& rng, const Aabb& bounds) {
  Pose frame;
  frame.R = random_rotation(rng);
  for (int a = 0; a < 3; ++a) frame.t[a] = uniform_range(rng, bounds.min[a], bounds.max[a]);
  return frame;
}

// neighbor_search.cpp:46-59
std::int32_t next_prime_at_least(std::int32_t n) {
  if (n <= 2) return 2;
  std::int32_t p = n | 1;
  for (;; p += 2) {
    bool prime = true;
    for (std::int32_t d = 3; d * d <= p; d += 2)
      if (p % d == 0) {
        prime = false;
        break;
      }
    if (prime) return p;
  }
}

namespace {
struct PassSetup {
  Pose frame;
  V6 noise;
  std::int32_t n_buckets;
  int idx_bits, h_bits, prio_bits;
  std::uint64_t idx_mask, prio_seed;
};
// neighbor_search.cpp:71-90
PassSetup pass_setup(std::size_t n, const LshConfig& cfg, std::uint64_t pass_seed, const Aabb& bounds) {
  PassSetup s;
  SplitMix64 rng(pass_seed);
  s.frame = random_lsh_frame(rng, bounds);
  const V6 z = normal6(rng);
  for (int c = 0; c < 6; ++c) s.noise[c] = cfg.noise_sigma * z[c];
  s.n_buckets = cfg.n_buckets > 0
                    ? cfg.n_buckets
                    : next_prime_at_least(static_cast<std::int32_t>(std::ceil(cfg.buckets_factor * static_cast<double>(n))));
  s.idx_bits = std::max(1, static_cast<int>(std::bit_width(n - 1)));
  s.h_bits = std::max(1, static_cast<int>(std::bit_width(static_cast<std::uint32_t>(s.n_buckets - 1))));
  s.prio_bits = std::max(0, 64 - s.h_bits - s.idx_bits);
  s.idx_mask = (std::uint64_t(1) << s.idx_bits) - 1;
  s.prio_seed = mix_seed(pass_seed, 0x70726f6974ull);
  return s;
}
inline std::uint64_t make_key(const PassSetup& s, const Pose& pose, std::size_t i, const LshConfig& cfg,
                              const KernelParams& kp) {
  const std::uint64_t h = lsh_hash(pose, s.frame, s.noise, cfg, kp) % static_cast<std::uint64_t>(s.n_buckets);
  const std::uint64_t prio = s.prio_bits > 0 ? mix_seed(s.prio_seed, static_cast<std::uint64_t>(i)) >> (64 - s.prio_bits) : 0;
  return (h << (s.prio_bits + s.idx_bits)) | (prio << s.idx_bits) | static_cast<std::uint64_t>(i);
}
}  // namespace

// neighbor_search.cpp:61-192
NeighborStats update_neighbors(ParticleSet& set, const LshConfig& cfg, const KernelParams& kp,
                               std::uint64_t pass_seed, const Aabb& bounds) {
  const std::size_t n = set.size();
  NeighborStats stats;
  if (n == 0) return stats;
  if (set.neighbors.size() != n || set.neighbors.k_max != cfg.k_neighbors)
    throw std::invalid_argument("update_neighbors: graph not initialized for this set");
  const PassSetup s = pass_setup(n, cfg, pass_seed, bounds);
  stats.n_buckets = s.n_buckets;

  std::vector<std::uint64_t> keys(n);
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i)
    keys[static_cast<std::size_t>(i)] = make_key(s, set.poses[static_cast<std::size_t>(i)], static_cast<std::size_t>(i), cfg, kp);
  std::sort(keys.begin(), keys.end());  // unique keys: any correct sort gives this order

  std::vector<std::int32_t> member_of(n);
  for (std::size_t p = 0; p < n; ++p) member_of[p] = static_cast<std::int32_t>(keys[p] & s.idx_mask);
  if (cfg.reorder_particles) {
    set.reorder(member_of);
    std::iota(member_of.begin(), member_of.end(), 0);
  }
  const int shift = s.prio_bits + s.idx_bits;
  std::vector<std::int32_t> run_begin(n), run_end(n);
  for (std::size_t p = 0; p < n; ++p)
    run_begin[p] = (p > 0 && (keys[p] >> shift) == (keys[p - 1] >> shift)) ? run_begin[p - 1] : static_cast<std::int32_t>(p);
  for (std::size_t p = n; p-- > 0;)
    run_end[p] = (p + 1 < n && (keys[p] >> shift) == (keys[p + 1] >> shift)) ? run_end[p + 1] : static_cast<std::int32_t>(p + 1);

  auto& graph = set.neighbors;
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) graph.refresh(static_cast<std::size_t>(i), set.poses, kp);

#pragma omp parallel for schedule(dynamic, 1024)
  for (std::int64_t p = 0; p < static_cast<std::int64_t>(n); ++p) {
    const std::int32_t i = member_of[static_cast<std::size_t>(p)];
    const std::int32_t begin = run_begin[static_cast<std::size_t>(p)];
    const std::int32_t end = std::min(run_end[static_cast<std::size_t>(p)], begin + cfg.bucket_capacity);
    const Pose& pi = set.poses[static_cast<std::size_t>(i)];
    const Pose inv_i = inverse(pi);
    for (std::int32_t q = begin; q < end; ++q) {
      const std::int32_t j = member_of[static_cast<std::size_t>(q)];
      if (j == i) continue;
      float k_ij = 0.0f;
      if (!kernel_underflows(pi, set.poses[static_cast<std::size_t>(j)], kp))
        k_ij = static_cast<float>(kernel_of_tangent(se3_log(compose(inv_i, set.poses[static_cast<std::size_t>(j)])), kp));
      graph.offer(static_cast<std::size_t>(i), j, k_ij);
    }
  }

  stats.occupancy_hist.assign(static_cast<std::size_t>(cfg.bucket_capacity) + 2, 0);
  for (std::size_t p = 0; p < n;) {
    const std::int64_t size = run_end[p] - run_begin[p];
    ++stats.buckets_used;
    ++stats.occupancy_hist[std::min<std::size_t>(static_cast<std::size_t>(size), stats.occupancy_hist.size() - 1)];
    if (size > cfg.bucket_capacity) stats.overflow_dropped += size - cfg.bucket_capacity;
    p = static_cast<std::size_t>(run_end[p]);
  }
  const double kernel_sum = chunked_sum(n, [&](std::size_t i) {
    double acc = 0.0;
    const std::size_t base = i * static_cast<std::size_t>(graph.k_max);
    for (int s2 = 0; s2 < graph.count[i]; ++s2) acc += graph.kval[base + static_cast<std::size_t>(s2)];
    return acc;
  });
  const double entries = chunked_sum(n, [&](std::size_t i) { return static_cast<double>(graph.count[i]); });
  stats.mean_kernel = entries > 0 ? kernel_sum / entries : 0.0;
  return stats;
}

// reference.cpp:78-167 (serial twin: plain loop over bucket runs).
NeighborStats update_neighbors_serial(ParticleSet& set, const LshConfig& cfg, const KernelParams& kp,
                                      std::uint64_t pass_seed, const Aabb& bounds) {
  const std::size_t n = set.size();
  NeighborStats stats;
  if (n == 0) return stats;
  const PassSetup s = pass_setup(n, cfg, pass_seed, bounds);
  stats.n_buckets = s.n_buckets;
  std::vector<std::uint64_t> keys(n);
  for (std::size_t i = 0; i < n; ++i) keys[i] = make_key(s, set.poses[i], i, cfg, kp);
  std::sort(keys.begin(), keys.end());
  std::vector<std::int32_t> member_of(n);
  for (std::size_t p = 0; p < n; ++p) member_of[p] = static_cast<std::int32_t>(keys[p] & s.idx_mask);
  if (cfg.reorder_particles) {
    set.reorder(member_of);
    std::iota(member_of.begin(), member_of.end(), 0);
  }
  for (std::size_t i = 0; i < n; ++i) set.neighbors.refresh(i, set.poses, kp);
  const int shift = s.prio_bits + s.idx_bits;
  stats.occupancy_hist.assign(static_cast<std::size_t>(cfg.bucket_capacity) + 2, 0);
  std::size_t run_begin = 0;
  while (run_begin < n) {
    std::size_t run_end = run_begin + 1;
    while (run_end < n && (keys[run_end] >> shift) == (keys[run_begin] >> shift)) ++run_end;
    const std::size_t visible_end = std::min(run_end, run_begin + static_cast<std::size_t>(cfg.bucket_capacity));
    for (std::size_t p = run_begin; p < run_end; ++p) {
      const std::int32_t i = member_of[p];
      const Pose inv_i = inverse(set.poses[static_cast<std::size_t>(i)]);
      for (std::size_t q = run_begin; q < visible_end; ++q) {
        const std::int32_t j = member_of[q];
        if (j == i) continue;
        float k_ij = 0.0f;
        if (!kernel_underflows(set.poses[static_cast<std::size_t>(i)], set.poses[static_cast<std::size_t>(j)], kp))
          k_ij = static_cast<float>(kernel_of_tangent(se3_log(compose(inv_i, set.poses[static_cast<std::size_t>(j)])), kp));
        set.neighbors.offer(static_cast<std::size_t>(i), j, k_ij);
      }
    }
    const std::size_t size = run_end - run_begin;
    ++stats.buckets_used;
    ++stats.occupancy_hist[std::min(size, stats.occupancy_hist.size() - 1)];
    if (size > static_cast<std::size_t>(cfg.bucket_capacity))
      stats.overflow_dropped += static_cast<std::int64_t>(size) - cfg.bucket_capacity;
    run_begin = run_end;
  }
  double kernel_sum = 0.0, entries = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    for (int s2 = 0; s2 < set.neighbors.count[i]; ++s2)
      kernel_sum += set.neighbors.kval[i * static_cast<std::size_t>(set.neighbors.k_max) + static_cast<std::size_t>(s2)];
    entries += static_cast<double>(set.neighbors.count[i]);
  }
  stats.mean_kernel = entries > 0 ? kernel_sum / entries : 0.0;
  return stats;
}

// reference.cpp:192-215 (recall oracle)
std::vector<std::vector<std::int32_t>> brute_force_kernel_knn(std::span<const Pose> poses, int k,
                                                              const KernelParams& kp) {
  const std::size_t n = poses.size();
  std::vector<std::vector<std::int32_t>> out(n);
#pragma omp parallel
  {
    std::vector<std::pair<double, std::int32_t>> cand(n);
#pragma omp for schedule(static)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
      const Pose inv_i = inverse(poses[static_cast<std::size_t>(i)]);
      for (std::size_t j = 0; j < n; ++j) {
        const double kv = j == static_cast<std::size_t>(i) ? 1.0 : kernel_of_tangent(se3_log(compose(inv_i, poses[j])), kp);
        cand[j] = {-kv, static_cast<std::int32_t>(j)};
      }
      const std::size_t keep = std::min<std::size_t>(static_cast<std::size_t>(k), n);
      std::partial_sort(cand.begin(), cand.begin() + static_cast<std::ptrdiff_t>(keep), cand.end());
      auto& list = out[static_cast<std::size_t>(i)];
      for (std::size_t s2 = 0; s2 < keep; ++s2) list.push_back(cand[s2].second);
    }
  }
  return out;
}

// ---------------------------------------------------------------- SVGD
// svgd.hpp:53-60
V6 kernel_grad(const Pose& a, const Pose& b, const KernelParams& kp) {
  const V6 d = se3_log(compose(inverse(a), b));
  const double k = kernel_of_tangent(d, kp);
  V6 g;
  for (int c = 0; c < 3; ++c) {
    g[c] = ((-2.0 * k) * kp.sigma_r) * d[c];
    g[c + 3] = ((-2.0 * k) * kp.sigma_t) * d[c + 3];
  }
  return g;
}

// svgd.cpp:7-34
V6 compute_phi(std::int32_t i, std::span<const Pose> poses, std::span<const V6> steps,
               std::span<const std::int32_t> nbrs, const KernelParams& kp) {
  const Pose& pi = poses[static_cast<std::size_t>(i)];
  const Pose inv_i = inverse(pi);
  V6 numer;
  double denom = 0.0;
  for (const std::int32_t j : nbrs) {
    const V6& sj = steps[static_cast<std::size_t>(j)];
    if (j == i) {
      for (int c = 0; c < 6; ++c) numer[c] = numer[c] + sj[c];
      denom += 1.0;
      continue;
    }
    const Pose& pj = poses[static_cast<std::size_t>(j)];
    if (kernel_underflows(pi, pj, kp)) continue;
    const V6 d = se3_log(compose(inv_i, pj));
    const double k = kernel_of_tangent(d, kp);
    const double gr = (-2.0 * k) * kp.sigma_r, gt = (-2.0 * k) * kp.sigma_t;
    for (int c = 0; c < 6; ++c) {
      const double grad = (c < 3 ? gr : gt) * d[c];
      numer[c] = numer[c] + (k * sj[c] + kp.repulsion_gain * grad);
    }
    denom += k;
  }
  V6 phi;
  for (int c = 0; c < 6; ++c) phi[c] = numer[c] / denom;
  return phi;
}

// svgd.cpp:36-49
void compute_phis(std::span<const Pose> poses, std::span<const V6> steps,
                  std::span<const std::int32_t> idx, std::span<const std::int32_t> count, int k_stride,
                  const KernelParams& kp, std::span<V6> phi_out, bool serial) {
  const std::int64_t n = static_cast<std::int64_t>(poses.size());
#pragma omp parallel for schedule(static) if (!serial)
  for (std::int64_t i = 0; i < n; ++i) {
    const std::size_t base = static_cast<std::size_t>(i) * static_cast<std::size_t>(k_stride);
    phi_out[static_cast<std::size_t>(i)] =
        compute_phi(static_cast<std::int32_t>(i), poses, steps,
                    idx.subspan(base, static_cast<std::size_t>(count[static_cast<std::size_t>(i)])), kp);
  }
}

// svgd.cpp:51-62
void apply_updates(std::span<Pose> poses, std::span<const V6> phis, bool serial) {
  if (poses.size() != phis.size()) throw std::invalid_argument("apply_updates: one phi per particle required");
  const std::int64_t n = static_cast<std::int64_t>(poses.size());
#pragma omp parallel for schedule(static) if (!serial)
  for (std::int64_t i = 0; i < n; ++i) {
    Pose& p = poses[static_cast<std::size_t>(i)];
    p = compose(p, se3_exp(phis[static_cast<std::size_t>(i)]));
    renormalize_if_needed(p);
  }
}

}  // namespace orc
