// ORACLE — test infrastructure only. Posterior and filter orchestration
// restated from /root/reference/proj/src/posterior.cpp:13-108 and
// src/filter.cpp:25-213 (with reference.cpp:169-190 for the serial smooth).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <stdexcept>

#include "oracle.hpp"

namespace orc {

// ---------------------------------------------------------------- posterior
void normalize_log_post(std::span<double> log_post, double floor) {  // posterior.cpp:13-24
  const std::size_t n = log_post.size();
  if (n == 0) return;
  const double m = chunked_argmax(n, [&](std::size_t i) { return log_post[i]; }).value;
  const double sum = chunked_sum(n, [&](std::size_t i) { return std::exp(log_post[i] - m); });
  const double lse = m + std::log(sum);
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    double& v = log_post[static_cast<std::size_t>(i)];
    v = std::max(v - lse, floor);
  }
}

bool bayes_update(std::span<double> log_post, std::span<const double> ll, std::span<const std::int32_t> nm,
                  double beta, double floor) {  // posterior.cpp:26-58
  if (!(beta >= 0.0)) throw std::invalid_argument("bayes_update: beta must be >= 0");
  const std::size_t n = log_post.size();
  if (ll.size() != n || nm.size() != n) throw std::invalid_argument("bayes_update: size mismatch");
  if (n == 0) return false;
  const double matched = chunked_sum(n, [&](std::size_t i) { return ll[i] > k_unmatched_log_lik ? 1.0 : 0.0; });
  if (matched == 0.0) {
    const double uniform = -std::log(static_cast<double>(n));
    for (std::size_t i = 0; i < n; ++i) log_post[i] = uniform;
    return true;
  }
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    const std::size_t k = static_cast<std::size_t>(i);
    const double denom = std::max(nm[k], 1);
    log_post[k] += beta * ll[k] / denom;
  }
  normalize_log_post(log_post, floor);
  return false;
}

void smooth(std::span<double> log_post, const NeighborGraph& g, int iters, double floor, bool serial) {  // 60-97
  if (iters < 0) throw std::invalid_argument("smooth: iters must be >= 0");
  const std::size_t n = log_post.size();
  if (n == 0 || iters == 0) return;
  if (g.size() != n) throw std::invalid_argument("smooth: graph size mismatch");
  std::vector<double> p(n), q(n);
#pragma omp parallel for schedule(static) if (!serial)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i)
    p[static_cast<std::size_t>(i)] = std::exp(log_post[static_cast<std::size_t>(i)]);
  for (int round = 0; round < iters; ++round) {
#pragma omp parallel for schedule(static) if (!serial)
    for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
      const std::size_t k = static_cast<std::size_t>(i);
      const std::size_t base = k * static_cast<std::size_t>(g.k_max);
      double num = 0.0, den = 0.0;
      for (int s = 0; s < g.count[k]; ++s) {
        const double w = g.kval[base + static_cast<std::size_t>(s)];
        num += w * p[static_cast<std::size_t>(g.idx[base + static_cast<std::size_t>(s)])];
        den += w;
      }
      q[k] = num / den;
    }
    p.swap(q);
  }
#pragma omp parallel for schedule(static) if (!serial)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i)
    log_post[static_cast<std::size_t>(i)] = std::log(p[static_cast<std::size_t>(i)]);
  normalize_log_post(log_post, floor);
}

ArgMax representative(std::span<const double> log_post) {  // posterior.cpp:99-108
  if (log_post.empty()) throw std::invalid_argument("representative: empty or mismatched particle set");
  return chunked_argmax(log_post.size(), [&](std::size_t i) { return log_post[i]; });
}

// ---------------------------------------------------------------- filter
namespace {
enum : std::uint64_t { k_stream_init = 1, k_stream_predict = 2, k_stream_neighbors = 3 };  // filter.cpp:22-23
using Clock = std::chrono::steady_clock;
double ms_since(const Clock::time_point& t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

bool llt6(const M6& a, M6& l) {  // Eigen LLT lower, unblocked
  l = a;
  for (int k = 0; k < 6; ++k) {
    double x = l(k, k);
    if (k > 0) {
      double sq = 0.0;
      for (int j = 0; j < k; ++j) sq += l(k, j) * l(k, j);
      x -= sq;
    }
    if (x <= 0.0) return false;
    x = std::sqrt(x);
    l(k, k) = x;
    for (int i = k + 1; i < 6; ++i) {
      if (k > 0) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s += l(i, j) * l(k, j);
        l(i, k) -= s;
      }
      l(i, k) /= x;
    }
  }
  for (int i = 0; i < 6; ++i)
    for (int j = i + 1; j < 6; ++j) l(i, j) = 0.0;
  return true;
}

// Symmetric 6x6 Jacobi eigen-decomposition (stand-in for Eigen's
// SelfAdjointEigenSolver in the rank-deficient covariance_sqrt fallback).
void sym_eig6(const M6& a_in, double w[6], M6& v) {
  M6 a = a_in;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) v(i, j) = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, scale = 0.0;
    for (int i = 0; i < 6; ++i) {
      scale += std::fabs(a(i, i));
      for (int j = i + 1; j < 6; ++j) off += std::fabs(a(i, j));
    }
    if (off == 0.0 || off < 1e-18 * scale) break;
    for (int p = 0; p < 5; ++p)
      for (int q = p + 1; q < 6; ++q) {
        if (a(p, q) == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 6; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < 6; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < 6; ++k) {
          const double vkp = v(k, p), vkq = v(k, q);
          v(k, p) = c * vkp - s * vkq;
          v(k, q) = s * vkp + c * vkq;
        }
      }
  }
  // Ascending order, as Eigen's SelfAdjointEigenSolver returns them.
  int ord[6] = {0, 1, 2, 3, 4, 5};
  std::sort(ord, ord + 6, [&](int x, int y) { return a(x, x) < a(y, y); });
  M6 vs;
  for (int c = 0; c < 6; ++c) {
    w[c] = a(ord[c], ord[c]);
    for (int r = 0; r < 6; ++r) vs(r, c) = v(r, ord[c]);
  }
  v = vs;
}
}  // namespace

M6 covariance_sqrt(const M6& cov) {  // filter.cpp:25-35
  M6 l;
  if (llt6(cov, l)) return l;
  M6 jit = cov;
  for (int i = 0; i < 6; ++i) jit(i, i) = cov(i, i) + 1e-12;
  if (llt6(jit, l)) return l;
  double w[6];
  M6 v;
  sym_eig6(cov, w, v);
  M6 out;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) out(i, j) = v(i, j) * std::sqrt(std::max(w[j], 0.0));
  return out;
}

// filter.cpp:39-65
ParticleSet init_uniform(const FilterConfig& cfg, const Aabb& bounds, bool full_rotation, std::uint64_t seed) {
  if (cfg.n_particles < 1) throw std::invalid_argument("init_uniform: n_particles must be >= 1");
  for (int a = 0; a < 3; ++a)
    if (bounds.max[a] - bounds.min[a] <= 0.0) throw std::invalid_argument("init_uniform: degenerate bounds");
  const std::size_t n = static_cast<std::size_t>(cfg.n_particles);
  ParticleSet set;
  set.poses.resize(n);
  set.log_post.assign(n, -std::log(static_cast<double>(n)));
  set.id.resize(n);
  set.neighbors.init_self(n, cfg.lsh.k_neighbors);
  const std::uint64_t stream = mix_seed(seed, k_stream_init);
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    SplitMix64 rng(mix_seed(stream, static_cast<std::uint64_t>(i)));
    Pose& p = set.poses[static_cast<std::size_t>(i)];
    p.R = full_rotation ? random_rotation(rng) : random_yaw(rng);
    for (int a = 0; a < 3; ++a) p.t[a] = uniform_range(rng, bounds.min[a], bounds.max[a]);
    set.id[static_cast<std::size_t>(i)] = static_cast<std::int32_t>(i);
  }
  return set;
}

// filter.cpp:67-84
void predict(ParticleSet& set, const Pose& delta, const M6& cov, std::uint64_t frame_seed) {
  const std::size_t n = set.size();
  bool noiseless = true;
  for (double c : cov.m)
    if (c != 0.0) noiseless = false;
  const M6 sqrt_cov = noiseless ? M6{} : covariance_sqrt(cov);
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(n); ++i) {
    Pose& p = set.poses[static_cast<std::size_t>(i)];
    p = compose(p, delta);
    if (!noiseless) {
      SplitMix64 rng(mix_seed(frame_seed, static_cast<std::uint64_t>(i)));
      const V6 z = normal6(rng);
      V6 noise;
      for (int r = 0; r < 6; ++r) {
        double acc = sqrt_cov(r, 0) * z[0];
        for (int c = 1; c < 6; ++c) acc = acc + sqrt_cov(r, c) * z[c];
        noise[r] = acc;
      }
      p = compose(p, se3_exp(noise));
    }
    renormalize_if_needed(p);
  }
}

// filter.cpp:86-100
GaussianCloud make_scan_cloud(std::span<const V3> points, const FilterConfig& cfg) {
  if (points.size() < static_cast<std::size_t>(cfg.covariance_k) + 1 || points.size() < 5) return {};
  const std::vector<V3> down = downsample_to(points, static_cast<std::size_t>(cfg.n_scan_max), cfg.scan_voxel_leaf);
  const int k = std::min<int>(cfg.covariance_k, static_cast<int>(down.size()) - 1);
  if (k < 4) return {};
  GaussianCloud scan = estimate_covariances(down, k, cfg.epsilon_plane);
  const double noise_var = cfg.sensor_noise_sigma * cfg.sensor_noise_sigma;
  if (noise_var > 0.0)
    for (M3& s : scan.sigma)
      for (int d = 0; d < 3; ++d) s(d, d) = s(d, d) + noise_var;
  return scan;
}

FilterEngine::FilterEngine(GaussianCloud map, FilterConfig cfg) : map_(std::move(map)), cfg_(cfg) {  // 102-106
  if (map_.empty()) throw std::invalid_argument("FilterEngine: empty map");
  nnf_ = build_nnf(map_, cfg_.nnf_resolution, cfg_.nnf_padding, cfg_.nnf_max_query_dist);
}

void FilterEngine::init_uniform(const Aabb& bounds) {  // 108-116
  particles_ = orc::init_uniform(cfg_, bounds, cfg_.full_rotation, cfg_.seed);
  frame_ = 0;
  const std::size_t n = particles_.size();
  steps_.assign(n, V6{});
  phis_.assign(n, V6{});
  log_lik_.assign(n, 0.0);
  n_matched_.assign(n, 0);
}

// filter.cpp:118-213
FrameResult FilterEngine::step(const GaussianCloud& scan, const OdometryInput& odo) {
  if (particles_.size() == 0) throw std::logic_error("FilterEngine::step: not initialized");
  const auto t_total = Clock::now();
  const std::size_t n = particles_.size();
  FrameResult out;
  out.n_particles = n;
  out.scan_empty = scan.empty();

  auto t0 = Clock::now();
  {
    const Pose delta = odo.valid ? odo.delta : Pose{};
    M6 cov;
    if (odo.valid) {
      cov = odo.cov;
    } else {
      for (int d = 0; d < 3; ++d) {
        cov(d, d) = cfg_.diffusion_sigma_rot * cfg_.diffusion_sigma_rot;
        cov(d + 3, d + 3) = cfg_.diffusion_sigma_trans * cfg_.diffusion_sigma_trans;
      }
    }
    predict(particles_, delta, cov, mix_seed(cfg_.seed, k_stream_predict, static_cast<std::uint64_t>(frame_)));
  }
  out.times_ms[0] = ms_since(t0);

  t0 = Clock::now();
  out.neighbor_stats = update_neighbors(particles_, cfg_.lsh, cfg_.kernel,
                                        mix_seed(cfg_.seed, k_stream_neighbors, static_cast<std::uint64_t>(frame_)),
                                        map_.bounds);
  out.times_ms[1] = ms_since(t0);

  if (!scan.empty()) {
    const GaussianCloud* gn_scan = &scan;
    GaussianCloud strided;
    if (cfg_.gn_scan_stride > 1 && scan.size() > 2 * static_cast<std::size_t>(cfg_.gn_scan_stride)) {
      for (std::size_t k = 0; k < scan.size(); k += static_cast<std::size_t>(cfg_.gn_scan_stride)) {
        strided.mu.push_back(scan.mu[k]);
        strided.sigma.push_back(scan.sigma[k]);
      }
      strided.bounds = scan.bounds;
      gn_scan = &strided;
    }
    for (int iter = 0; iter < cfg_.n_svgd_iters; ++iter) {
      t0 = Clock::now();
      evaluate_all(map_, nnf_, *gn_scan, particles_.poses, cfg_.gicp, steps_, log_lik_, n_matched_);
      out.times_ms[2] += ms_since(t0);
      t0 = Clock::now();
      compute_phis(particles_.poses, steps_, particles_.neighbors.idx, particles_.neighbors.count,
                   particles_.neighbors.k_max, cfg_.kernel, phis_);
      apply_updates(particles_.poses, phis_);
      out.times_ms[3] += ms_since(t0);
    }
    t0 = Clock::now();
    evaluate_likelihoods(map_, nnf_, scan, particles_.poses, cfg_.gicp, log_lik_, n_matched_);
    out.times_ms[2] += ms_since(t0);
    t0 = Clock::now();
    out.observation_rejected = bayes_update(particles_.log_post, log_lik_, n_matched_, cfg_.beta, cfg_.log_post_floor);
    out.mean_n_matched = chunked_sum(n, [&](std::size_t i) { return double(n_matched_[i]); }) / static_cast<double>(n);
  } else {
    t0 = Clock::now();
  }
  smooth(particles_.log_post, particles_.neighbors, cfg_.smooth_iters, cfg_.log_post_floor);
  const ArgMax rep = representative(particles_.log_post);
  out.times_ms[4] = ms_since(t0);
  out.representative = particles_.poses[static_cast<std::size_t>(rep.index)];
  out.rep_log_post = rep.value;
  out.rep_index = rep.index;
  out.rep_id = particles_.id[static_cast<std::size_t>(rep.index)];
  out.times_ms[5] = ms_since(t_total);
  ++frame_;
  return out;
}

}  // namespace orc
