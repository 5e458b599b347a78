// steinmcl/b200.hpp — source-compatible `steinmcl::` facade over the C ABI
// (smcl_gpu.h, libsmcl_gpu.so). A reference call site compiles against it by
// putting this repo's include/ first on the include path: the header names
// (steinmcl/filter.hpp, gicp.hpp, neighbor_search.hpp, svgd.hpp,
// posterior.hpp, nnf.hpp, particle_set.hpp, neighbor_graph.hpp, se3.hpp,
// gaussian_cloud.hpp) forward here.
//
// Reference API mirrored (all paths /root/reference/proj/include/steinmcl/):
//   FilterConfig{kernel, lsh, gicp, ...}  filter.hpp:17-51
//   OdometryInput / StageTimes / FrameResult  filter.hpp:53-82
//   FilterEngine (map(), nnf(), particles(), mutable_particles(), config(),
//     frame_index())  filter.hpp:104-130
//   init_uniform / predict / make_scan_cloud  filter.hpp:84-102
//   GnSystem / StepLimits / GicpParams / solve_step / evaluate_all /
//     evaluate_likelihoods  gicp.hpp:18-72
//   LshConfig / NeighborStats / lsh_hash / update_neighbors /
//     next_prime_at_least  neighbor_search.hpp:13-48
//   KernelParams / compute_phis / apply_updates  svgd.hpp:13-81
//   normalize_log_post / bayes_update / smooth / representative  posterior.hpp:12-41
//   NearestNeighborField / build_nnf  nnf.hpp:13-50
//   ParticleSet / NeighborGraph  particle_set.hpp:16-27, neighbor_graph.hpp:16-90
//
// Linear algebra types. Without Eigen (this image has none) Vec3 / Mat3 /
// Vec6 / Mat6 are small value types with the Eigen accessors reference call
// sites use (x() y() z(), (i), (r, c), Zero(), Identity(), Constant(),
// transpose(), products). Define STEINMCL_B200_EIGEN (after including
// <Eigen/Core>) to make them the reference's Eigen types; the facade touches
// them only through (i) / (r, c), so both spellings compile.
//
// Stage functions run on the B200 through a transient engine on the current
// device (the particle state is uploaded, the stage runs, results come back),
// so they keep the reference's stateless host signatures. The hot path is
// FilterEngine::step, whose state stays resident in HBM between frames.
// Errors are rethrown as the exception types the reference throws.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "smcl_gpu.h"

#ifdef STEINMCL_B200_EIGEN
#include <Eigen/Core>
#endif

namespace steinmcl {

// ------------------------------------------------------------------ algebra
#ifdef STEINMCL_B200_EIGEN
using Vec3 = Eigen::Vector3d;
using Mat3 = Eigen::Matrix3d;
using Vec6 = Eigen::Matrix<double, 6, 1>;
using Mat6 = Eigen::Matrix<double, 6, 6>;
#else
template <int N>
struct Vec {
  double v[N] = {};
  Vec() = default;
  template <class... T>
    requires(sizeof...(T) == N && N > 1)
  Vec(T... a) : v{static_cast<double>(a)...} {}
  static Vec Zero() { return Vec(); }
  static Vec Constant(double c) {
    Vec r;
    for (int i = 0; i < N; ++i) r.v[i] = c;
    return r;
  }
  double& operator()(int i) { return v[i]; }
  double operator()(int i) const { return v[i]; }
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
  double& x() { return v[0]; }
  double& y() { return v[1]; }
  double& z() { return v[2]; }
  double x() const { return v[0]; }
  double y() const { return v[1]; }
  double z() const { return v[2]; }
  static constexpr int size() { return N; }
  double dot(const Vec& o) const {
    double s = 0.0;
    for (int i = 0; i < N; ++i) s += v[i] * o.v[i];
    return s;
  }
  double squaredNorm() const { return dot(*this); }
  double norm() const { return std::sqrt(squaredNorm()); }
  Vec operator+(const Vec& o) const {
    Vec r;
    for (int i = 0; i < N; ++i) r.v[i] = v[i] + o.v[i];
    return r;
  }
  Vec operator-(const Vec& o) const {
    Vec r;
    for (int i = 0; i < N; ++i) r.v[i] = v[i] - o.v[i];
    return r;
  }
  Vec operator-() const { return Vec() - *this; }
  Vec operator*(double s) const {
    Vec r;
    for (int i = 0; i < N; ++i) r.v[i] = v[i] * s;
    return r;
  }
  friend Vec operator*(double s, const Vec& a) { return a * s; }
  Vec& operator+=(const Vec& o) { return *this = *this + o; }
  Vec& operator-=(const Vec& o) { return *this = *this - o; }
  bool operator==(const Vec& o) const {
    for (int i = 0; i < N; ++i)
      if (v[i] != o.v[i]) return false;
    return true;
  }
};
template <int N>
struct Mat {  // row-major storage; access through (r, c) only
  double m[N * N] = {};
  static Mat Zero() { return Mat(); }
  static Mat Identity() {
    Mat r;
    for (int i = 0; i < N; ++i) r.m[i * N + i] = 1.0;
    return r;
  }
  double& operator()(int r, int c) { return m[r * N + c]; }
  double operator()(int r, int c) const { return m[r * N + c]; }
  static constexpr int rows() { return N; }
  static constexpr int cols() { return N; }
  Mat transpose() const {
    Mat t;
    for (int r = 0; r < N; ++r)
      for (int c = 0; c < N; ++c) t.m[c * N + r] = m[r * N + c];
    return t;
  }
  Mat operator*(const Mat& o) const {
    Mat p;
    for (int r = 0; r < N; ++r)
      for (int c = 0; c < N; ++c) {
        double s = 0.0;
        for (int k = 0; k < N; ++k) s += m[r * N + k] * o.m[k * N + c];
        p.m[r * N + c] = s;
      }
    return p;
  }
  Vec<N> operator*(const Vec<N>& x) const {
    Vec<N> y;
    for (int r = 0; r < N; ++r) {
      double s = 0.0;
      for (int k = 0; k < N; ++k) s += m[r * N + k] * x.v[k];
      y.v[r] = s;
    }
    return y;
  }
  Mat operator+(const Mat& o) const {
    Mat r;
    for (int i = 0; i < N * N; ++i) r.m[i] = m[i] + o.m[i];
    return r;
  }
  Mat operator*(double s) const {
    Mat r;
    for (int i = 0; i < N * N; ++i) r.m[i] = m[i] * s;
    return r;
  }
  friend Mat operator*(double s, const Mat& a) { return a * s; }
};
using Vec3 = Vec<3>;
using Mat3 = Mat<3>;
using Vec6 = Vec<6>;
using Mat6 = Mat<6>;
#endif
using Tangent = Vec6;  // [omega; v] (se3.hpp:15-17)

// Rigid transform, perturbations right-multiplied (se3.hpp:30-59).
struct Pose {
  Mat3 R = Mat3::Identity();
  Vec3 t = Vec3::Zero();
  static Pose identity() { return {}; }
  Pose inverse() const {
    Pose p;
    p.R = R.transpose();
    p.t = -(p.R * t);
    return p;
  }
};
inline Pose operator*(const Pose& a, const Pose& b) {  // se3.hpp:61-66
  Pose c;
  c.R = a.R * b.R;
  c.t = a.R * b.t + a.t;
  return c;
}
inline Vec3 operator*(const Pose& a, const Vec3& p) { return a.R * p + a.t; }

// Counter-seeded streams (rng.hpp:15-43): the seeds FilterEngine::step
// derives per stage and frame.
struct SplitMix64 {
  std::uint64_t state = 0;
  SplitMix64() = default;
  explicit SplitMix64(std::uint64_t seed) : state(seed) {}
  using result_type = std::uint64_t;
  static constexpr std::uint64_t min() { return 0; }
  static constexpr std::uint64_t max() { return ~std::uint64_t(0); }
  std::uint64_t operator()() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
};
inline std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b) {
  SplitMix64 g(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
  return g();
}
inline std::uint64_t mix_seed(std::uint64_t a, std::uint64_t b, std::uint64_t c) { return mix_seed(mix_seed(a, b), c); }

// ------------------------------------------------------------------ clouds and map
struct Aabb {  // gaussian_cloud.hpp:21-31
  Vec3 min = Vec3::Zero();
  Vec3 max = Vec3::Zero();
  Vec3 extent() const { return max - min; }
  Vec3 center() const { return 0.5 * (min + max); }
  bool contains(const Vec3& p) const {
    for (int a = 0; a < 3; ++a)
      if (!(p(a) >= min(a) && p(a) <= max(a))) return false;
    return true;
  }
  Aabb padded(double pad) const { return {min - Vec3::Constant(pad), max + Vec3::Constant(pad)}; }
};

struct PointGaussian {
  Vec3 mu;
  Mat3 sigma;
};

struct GaussianCloud {  // gaussian_cloud.hpp:32-40
  std::vector<Vec3> mu;
  std::vector<Mat3> sigma;
  Aabb bounds;
  std::size_t size() const { return mu.size(); }
  bool empty() const { return mu.empty(); }
  PointGaussian point(std::size_t i) const { return {mu[i], sigma[i]}; }
};

struct NearestNeighborField {  // nnf.hpp:13-35 (+ padding: the build argument)
  static constexpr std::int32_t k_empty = -1;
  Vec3 origin = Vec3::Zero();
  double resolution = 0.1;
  double max_query_dist = 1.0;
  double padding = 0.5;
  std::int32_t dims[3] = {0, 0, 0};
  std::vector<std::int32_t> cells;
  std::int32_t lookup_nearest(const Vec3& p) const {
    const double inv = 1.0 / resolution;
    const int x = static_cast<int>(std::floor((p.x() - origin.x()) * inv));
    const int y = static_cast<int>(std::floor((p.y() - origin.y()) * inv));
    const int z = static_cast<int>(std::floor((p.z() - origin.z()) * inv));
    if (static_cast<unsigned>(x) >= static_cast<unsigned>(dims[0]) ||
        static_cast<unsigned>(y) >= static_cast<unsigned>(dims[1]) ||
        static_cast<unsigned>(z) >= static_cast<unsigned>(dims[2]))
      return k_empty;
    return cells[(static_cast<std::size_t>(z) * dims[1] + y) * dims[0] + x];
  }
  std::size_t cell_count() const { return cells.size(); }
};

// ------------------------------------------------------------------ parameters
struct KernelParams {  // svgd.hpp:13-26
  double sigma_r = 5.0;
  double sigma_t = 2.5;
  double repulsion_gain = 1.0;
};
struct LshConfig {  // neighbor_search.hpp:13-21
  double alpha = 0.1;
  double noise_sigma = 0.5;
  double buckets_factor = 2.0;
  int n_buckets = 0;
  int bucket_capacity = 64;
  int k_neighbors = 20;
  bool reorder_particles = true;
};
struct StepLimits {  // gicp.hpp:33-36
  double omega_max = 0.5;
  double v_max = 1.0;
};
struct GicpParams {  // gicp.hpp:41-46
  double damping_scale = 1e-3;
  StepLimits limits;
  double min_match_fraction = 0.5;
  double miss_cost = 25.0;
};
inline constexpr double k_unmatched_log_lik = -1e30;
inline constexpr double k_default_log_post_floor = -80.0;

struct FilterConfig {  // filter.hpp:17-51
  int n_particles = 10000;
  KernelParams kernel;
  LshConfig lsh;
  double nnf_resolution = 0.1;
  double nnf_max_query_dist = 1.0;
  double nnf_padding = 0.5;
  int smooth_iters = 10;
  double beta = 2.0;
  int n_svgd_iters = 1;
  int gn_scan_stride = 1;
  GicpParams gicp;
  double log_post_floor = k_default_log_post_floor;
  int covariance_k = 10;
  double epsilon_plane = 1e-3;
  int n_scan_max = 1000;
  double scan_voxel_leaf = 0.05;
  double sensor_noise_sigma = 0.01;
  double diffusion_sigma_rot = 0.02;
  double diffusion_sigma_trans = 0.5;
  bool full_rotation = true;
  std::uint64_t seed = 1;
  // B200 extensions: likelihood arithmetic (0 auto, 1 exact fp64, 2 fast
  // structured fp32) and the CUDA device of the engine (< 0: current).
  int likelihood_mode = 0;
  int device = 0;
};

struct OdometryInput {  // filter.hpp:53-60
  Pose delta;
  Mat6 cov = Mat6::Zero();
  bool valid = true;
};

struct StageTimes {  // filter.hpp:62-69
  double predict_ms = 0.0;
  double neighbor_ms = 0.0;
  double likelihood_ms = 0.0;
  double update_ms = 0.0;
  double posterior_ms = 0.0;
  double total_ms = 0.0;
};

struct NeighborStats {  // neighbor_search.hpp:30-36
  std::int64_t n_buckets = 0;
  std::int64_t buckets_used = 0;
  std::int64_t overflow_dropped = 0;
  std::vector<std::int64_t> occupancy_hist;
  double mean_kernel = 0.0;
};

struct FrameResult {  // filter.hpp:71-82
  Pose representative;
  double rep_log_post = 0.0;
  std::int64_t rep_index = -1;
  std::int32_t rep_id = -1;
  std::size_t n_particles = 0;
  double mean_n_matched = 0.0;
  bool scan_empty = false;
  bool observation_rejected = false;
  NeighborStats neighbor_stats;
  StageTimes times;
};

struct GnSystem {  // gicp.hpp:18-23
  Mat6 H = Mat6::Zero();
  Vec6 b = Vec6::Zero();
  double log_lik = 0.0;
  int n_matched = 0;
};

struct Representative {  // posterior.hpp:33-37
  std::int64_t index = -1;
  Pose pose;
  double log_post = 0.0;
};

// ------------------------------------------------------------------ particles
struct NeighborGraph {  // neighbor_graph.hpp:16-45 (offer/refresh run on the device)
  int k_max = 20;
  std::vector<std::int32_t> idx;
  std::vector<float> kval;
  std::vector<std::int32_t> count;
  std::size_t size() const { return count.size(); }
  void init_self(std::size_t n, int k) {
    k_max = k;
    idx.assign(n * static_cast<std::size_t>(k), -1);
    kval.assign(n * static_cast<std::size_t>(k), 0.0f);
    count.assign(n, 1);
    for (std::size_t i = 0; i < n; ++i) {
      idx[i * static_cast<std::size_t>(k)] = static_cast<std::int32_t>(i);
      kval[i * static_cast<std::size_t>(k)] = 1.0f;
    }
  }
  std::span<const std::int32_t> neighbors_of(std::size_t i) const {
    return {idx.data() + i * static_cast<std::size_t>(k_max), static_cast<std::size_t>(count[i])};
  }
  std::span<const float> kernels_of(std::size_t i) const {
    return {kval.data() + i * static_cast<std::size_t>(k_max), static_cast<std::size_t>(count[i])};
  }
};

struct ParticleSet {  // particle_set.hpp:16-27
  std::vector<Pose> poses;
  std::vector<double> log_post;
  std::vector<std::int32_t> id;
  NeighborGraph neighbors;
  std::size_t size() const { return poses.size(); }
  // particle_set.cpp:7-47: slot p takes the particle at old_of_new[p],
  // neighbour indices remapped (a host permutation of host data).
  void reorder(std::span<const std::int32_t> old_of_new) {
    const std::size_t n = size(), k = static_cast<std::size_t>(neighbors.k_max);
    std::vector<std::int32_t> new_of_old(n);
    for (std::size_t p = 0; p < n; ++p) new_of_old[static_cast<std::size_t>(old_of_new[p])] = static_cast<std::int32_t>(p);
    ParticleSet o = *this;
    for (std::size_t p = 0; p < n; ++p) {
      const std::size_t s = static_cast<std::size_t>(old_of_new[p]);
      poses[p] = o.poses[s];
      log_post[p] = o.log_post[s];
      id[p] = o.id[s];
      neighbors.count[p] = o.neighbors.count[s];
      for (std::size_t q = 0; q < k; ++q) {
        const std::int32_t e = o.neighbors.idx[s * k + q];
        neighbors.idx[p * k + q] = e >= 0 ? new_of_old[static_cast<std::size_t>(e)] : e;
        neighbors.kval[p * k + q] = o.neighbors.kval[s * k + q];
      }
    }
  }
};

// ------------------------------------------------------------------ ABI plumbing
namespace b200 {
inline void check(int rc) {
  if (rc == SMCL_OK) return;
  const std::string msg = smcl_last_error();
  if (rc == SMCL_EINVAL) throw std::invalid_argument(msg);
  if (rc == SMCL_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

inline void pose_to12(const Pose& p, double* o) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) o[r * 3 + c] = p.R(r, c);
    o[9 + r] = p.t(r);
  }
}
inline Pose pose_from12(const double* o) {
  Pose p;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) p.R(r, c) = o[r * 3 + c];
    p.t(r) = o[9 + r];
  }
  return p;
}
inline void bounds_to6(const Aabb& b, double* o) {
  for (int a = 0; a < 3; ++a) {
    o[a] = b.min(a);
    o[3 + a] = b.max(a);
  }
}

inline smcl_config to_abi(const FilterConfig& c) {
  smcl_config a;
  smcl_config_default(&a);
  a.n_particles = c.n_particles;
  a.k_neighbors = c.lsh.k_neighbors;
  a.sigma_r = c.kernel.sigma_r;
  a.sigma_t = c.kernel.sigma_t;
  a.repulsion_gain = c.kernel.repulsion_gain;
  a.lsh_alpha = c.lsh.alpha;
  a.lsh_noise_sigma = c.lsh.noise_sigma;
  a.lsh_buckets_factor = c.lsh.buckets_factor;
  a.lsh_n_buckets = c.lsh.n_buckets;
  a.lsh_bucket_capacity = c.lsh.bucket_capacity;
  a.reorder_particles = c.lsh.reorder_particles ? 1 : 0;
  a.smooth_iters = c.smooth_iters;
  a.nnf_resolution = c.nnf_resolution;
  a.nnf_max_query_dist = c.nnf_max_query_dist;
  a.nnf_padding = c.nnf_padding;
  a.beta = c.beta;
  a.n_svgd_iters = c.n_svgd_iters;
  a.gn_scan_stride = c.gn_scan_stride;
  a.damping_scale = c.gicp.damping_scale;
  a.omega_max = c.gicp.limits.omega_max;
  a.v_max = c.gicp.limits.v_max;
  a.min_match_fraction = c.gicp.min_match_fraction;
  a.miss_cost = c.gicp.miss_cost;
  a.log_post_floor = c.log_post_floor;
  a.covariance_k = c.covariance_k;
  a.n_scan_max = c.n_scan_max;
  a.epsilon_plane = c.epsilon_plane;
  a.scan_voxel_leaf = c.scan_voxel_leaf;
  a.sensor_noise_sigma = c.sensor_noise_sigma;
  a.diffusion_sigma_rot = c.diffusion_sigma_rot;
  a.diffusion_sigma_trans = c.diffusion_sigma_trans;
  a.full_rotation = c.full_rotation ? 1 : 0;
  a.likelihood_mode = c.likelihood_mode;
  a.seed = c.seed;
  return a;
}

// Flat row-major copy of a cloud (+ bounds) kept alive for one ABI call.
struct CloudBuf {
  std::vector<double> mu, sigma;
  double b[6];
  smcl_cloud view{};
  explicit CloudBuf(const GaussianCloud& c, bool with_bounds = true) : mu(c.size() * 3), sigma(c.size() * 9) {
    for (std::size_t i = 0; i < c.size(); ++i)
      for (int r = 0; r < 3; ++r) {
        mu[3 * i + r] = c.mu[i](r);
        for (int q = 0; q < 3; ++q) sigma[9 * i + 3 * r + q] = c.sigma[i](r, q);
      }
    bounds_to6(c.bounds, b);
    view = smcl_cloud{static_cast<int64_t>(c.size()), mu.data(), sigma.data(), with_bounds ? b : nullptr};
  }
};

inline GaussianCloud cloud_from(const std::vector<double>& mu, const std::vector<double>& sigma, std::int64_t n) {
  GaussianCloud g;
  g.mu.resize(static_cast<std::size_t>(n));
  g.sigma.resize(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i)
    for (int r = 0; r < 3; ++r) {
      g.mu[static_cast<std::size_t>(i)](r) = mu[static_cast<std::size_t>(3 * i + r)];
      for (int q = 0; q < 3; ++q) g.sigma[static_cast<std::size_t>(i)](r, q) = sigma[static_cast<std::size_t>(9 * i + 3 * r + q)];
    }
  if (n > 0) {  // compute_bounds (gaussian_cloud.cpp)
    g.bounds.min = g.bounds.max = g.mu[0];
    for (const Vec3& p : g.mu)
      for (int a = 0; a < 3; ++a) {
        g.bounds.min(a) = std::min(g.bounds.min(a), p(a));
        g.bounds.max(a) = std::max(g.bounds.max(a), p(a));
      }
  }
  return g;
}

struct Engine {  // owning handle
  smcl_engine* h = nullptr;
  Engine() = default;
  Engine(const GaussianCloud* map, const smcl_config& cfg, int device) {
    if (map) {
      CloudBuf m(*map);
      check(smcl_create(&m.view, &cfg, device, &h));
    } else {
      check(smcl_create(nullptr, &cfg, device, &h));
    }
  }
  ~Engine() {
    if (h) smcl_destroy(h);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
};

inline void upload(smcl_engine* h, const ParticleSet& s) {
  const std::int64_t n = static_cast<std::int64_t>(s.size());
  const int k = s.neighbors.k_max;
  std::vector<double> poses(static_cast<std::size_t>(n) * 12);
  for (std::int64_t i = 0; i < n; ++i) pose_to12(s.poses[static_cast<std::size_t>(i)], &poses[static_cast<std::size_t>(12 * i)]);
  // Stage calls may pass a set without a graph or ids: fill self-only lists.
  std::vector<double> lp = s.log_post;
  std::vector<std::int32_t> id = s.id, idx = s.neighbors.idx, count = s.neighbors.count;
  std::vector<float> kval = s.neighbors.kval;
  lp.resize(static_cast<std::size_t>(n), n > 0 ? -std::log(static_cast<double>(n)) : 0.0);
  if (id.size() != static_cast<std::size_t>(n)) {
    id.resize(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) id[static_cast<std::size_t>(i)] = static_cast<std::int32_t>(i);
  }
  if (count.size() != static_cast<std::size_t>(n)) {
    NeighborGraph g;
    g.init_self(static_cast<std::size_t>(n), k);
    idx = g.idx;
    kval = g.kval;
    count = g.count;
  }
  smcl_particles_view v{n, k, poses.data(), lp.data(), id.data(), idx.data(), kval.data(), count.data()};
  check(smcl_set_particles(h, &v));
}

inline void download(smcl_engine* h, int k, ParticleSet& s) {
  const std::int64_t n = smcl_num_particles(h);
  std::vector<double> poses(static_cast<std::size_t>(n) * 12);
  s.log_post.resize(static_cast<std::size_t>(n));
  s.id.resize(static_cast<std::size_t>(n));
  s.neighbors.k_max = k;
  s.neighbors.idx.resize(static_cast<std::size_t>(n) * k);
  s.neighbors.kval.resize(static_cast<std::size_t>(n) * k);
  s.neighbors.count.resize(static_cast<std::size_t>(n));
  smcl_particles_view v{n, k, poses.data(), s.log_post.data(), s.id.data(), s.neighbors.idx.data(),
                        s.neighbors.kval.data(), s.neighbors.count.data()};
  check(smcl_get_particles(h, &v));
  s.poses.resize(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) s.poses[static_cast<std::size_t>(i)] = pose_from12(&poses[static_cast<std::size_t>(12 * i)]);
}

inline NeighborStats stats_from(const smcl_neighbor_stats& a) {
  NeighborStats s;
  s.n_buckets = a.n_buckets;
  s.buckets_used = a.buckets_used;
  s.overflow_dropped = a.overflow_dropped;
  s.mean_kernel = a.mean_kernel;
  s.occupancy_hist.assign(a.occupancy_hist, a.occupancy_hist + a.hist_len);
  return s;
}

inline FrameResult result_from(const smcl_frame_result& r) {
  FrameResult f;
  f.representative = pose_from12(r.representative);
  f.rep_log_post = r.rep_log_post;
  f.rep_index = r.rep_index;
  f.rep_id = r.rep_id;
  f.n_particles = static_cast<std::size_t>(r.n_particles);
  f.mean_n_matched = r.mean_n_matched;
  f.scan_empty = r.scan_empty != 0;
  f.observation_rejected = r.observation_rejected != 0;
  f.neighbor_stats = stats_from(r.neighbor_stats);
  f.times = {r.predict_ms, r.neighbor_ms, r.likelihood_ms, r.update_ms, r.posterior_ms, r.total_ms};
  return f;
}

inline smcl_odom odom_from(const OdometryInput& o) {
  smcl_odom a;
  pose_to12(o.delta, a.delta);
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) a.cov[r * 6 + c] = o.cov(r, c);
  a.valid = o.valid ? 1 : 0;
  return a;
}

// Transient engine holding (map, nnf) for the stateless likelihood stages.
// The NNF is rebuilt on the device from the map with the nnf's own
// parameters and must come out identical to the one passed in.
inline smcl_config map_stage_config(const NearestNeighborField& nnf, const GicpParams& gp, std::int64_t n) {
  FilterConfig c;
  c.n_particles = static_cast<int>(n > 0 ? n : 1);
  c.nnf_resolution = nnf.resolution;
  c.nnf_max_query_dist = nnf.max_query_dist;
  c.nnf_padding = nnf.padding;
  c.gicp = gp;
  return to_abi(c);
}
inline void check_nnf(smcl_engine* h, const NearestNeighborField& nnf) {
  int32_t dims[3];
  double origin[3], res = 0.0;
  check(smcl_get_nnf(h, dims, origin, &res, nullptr));
  for (int a = 0; a < 3; ++a)
    if (dims[a] != nnf.dims[a] || origin[a] != nnf.origin(a))
      throw std::invalid_argument("nnf was not built by build_nnf from this map");
}
inline std::vector<double> flat_poses(std::span<const Pose> poses) {
  std::vector<double> o(poses.size() * 12);
  for (std::size_t i = 0; i < poses.size(); ++i) pose_to12(poses[i], &o[12 * i]);
  return o;
}
inline void upload_poses(smcl_engine* h, std::span<const Pose> poses, int k = 1) {
  ParticleSet s;
  s.poses.assign(poses.begin(), poses.end());
  s.neighbors.k_max = k;
  upload(h, s);
}
}  // namespace b200

// ------------------------------------------------------------------ free functions
// build_nnf (nnf.cpp:10-96): built on the device by a transient engine.
inline NearestNeighborField build_nnf(const GaussianCloud& map, double resolution, double padding,
                                      double max_query_dist = 1.0, std::size_t max_cells = std::size_t(1) << 30) {
  if (map.empty()) throw std::invalid_argument("build_nnf: empty map");
  b200::CloudBuf m(map);
  NearestNeighborField f;
  f.resolution = resolution;
  f.max_query_dist = max_query_dist;
  f.padding = padding;
  double origin[3];
  b200::check(smcl_build_nnf(&m.view, resolution, padding, max_query_dist, f.dims, origin, nullptr));
  const std::size_t cells = static_cast<std::size_t>(f.dims[0]) * f.dims[1] * f.dims[2];
  if (cells > max_cells) throw std::runtime_error("build_nnf: cell count exceeds the memory budget");
  f.cells.resize(cells);
  b200::check(smcl_build_nnf(&m.view, resolution, padding, max_query_dist, f.dims, origin, f.cells.data()));
  for (int a = 0; a < 3; ++a) f.origin(a) = origin[a];
  return f;
}

// init_uniform(cfg, bounds, full_rotation, seed) (filter.cpp:39-65).
inline ParticleSet init_uniform(const FilterConfig& cfg, const Aabb& bounds, bool full_rotation, std::uint64_t seed) {
  b200::Engine e(nullptr, b200::to_abi(cfg), cfg.device);
  double b[6];
  b200::bounds_to6(bounds, b);
  b200::check(smcl_init_uniform_seeded(e.h, cfg.n_particles, b, full_rotation ? 1 : 0, seed));
  ParticleSet s;
  b200::download(e.h, cfg.lsh.k_neighbors, s);
  return s;
}

// predict(set, delta, cov, frame_seed) (filter.cpp:67-84).
inline void predict(ParticleSet& set, const Pose& delta, const Mat6& cov, std::uint64_t frame_seed) {
  FilterConfig c;
  c.n_particles = static_cast<int>(set.size());
  c.lsh.k_neighbors = set.neighbors.k_max;
  b200::Engine e(nullptr, b200::to_abi(c), -1);
  b200::upload(e.h, set);
  double d[12], cv[36];
  b200::pose_to12(delta, d);
  for (int r = 0; r < 6; ++r)
    for (int q = 0; q < 6; ++q) cv[r * 6 + q] = cov(r, q);
  b200::check(smcl_predict(e.h, d, cv, frame_seed));
  b200::download(e.h, set.neighbors.k_max, set);
}

// make_scan_cloud(points, cfg) (filter.cpp:86-100), host C++.
inline GaussianCloud make_scan_cloud(std::span<const Vec3> points, const FilterConfig& cfg) {
  std::vector<double> p(points.size() * 3);
  for (std::size_t i = 0; i < points.size(); ++i)
    for (int a = 0; a < 3; ++a) p[3 * i + a] = points[i](a);
  const smcl_config c = b200::to_abi(cfg);
  std::vector<double> mu(p.size()), sigma(points.size() * 9);
  int64_t m = 0;
  b200::check(smcl_make_scan_cloud(p.data(), static_cast<int64_t>(points.size()), &c, mu.data(), sigma.data(), &m));
  return b200::cloud_from(mu, sigma, m);
}

// lsh_hash(pose, frame, noise, cfg, kp) (neighbor_search.cpp:25-35), on the device.
inline std::uint64_t lsh_hash(const Pose& pose, const Pose& frame, const Vec6& noise, const LshConfig& cfg,
                              const KernelParams& kp) {
  double p[12], f[12], nz[6];
  b200::pose_to12(pose, p);
  b200::pose_to12(frame, f);
  for (int i = 0; i < 6; ++i) nz[i] = noise(i);
  uint64_t h = 0;
  b200::check(smcl_lsh_hash_batch(p, 1, f, nz, cfg.alpha, kp.sigma_r, kp.sigma_t, &h));
  return h;
}

inline std::int32_t next_prime_at_least(std::int32_t n) {  // neighbor_search.cpp:37-45
  auto prime = [](std::int64_t v) {
    if (v < 2) return false;
    for (std::int64_t d = 2; d * d <= v; ++d)
      if (v % d == 0) return false;
    return true;
  };
  std::int64_t v = n < 2 ? 2 : n;
  while (!prime(v)) ++v;
  return static_cast<std::int32_t>(v);
}

// update_neighbors(set, cfg, kp, pass_seed, bounds) (neighbor_search.cpp:61-192).
inline NeighborStats update_neighbors(ParticleSet& set, const LshConfig& cfg, const KernelParams& kp,
                                      std::uint64_t pass_seed, const Aabb& bounds) {
  if (set.neighbors.size() != set.size()) throw std::invalid_argument("update_neighbors: graph not initialized");
  FilterConfig c;
  c.n_particles = static_cast<int>(set.size());
  c.lsh = cfg;
  c.lsh.k_neighbors = set.neighbors.k_max;
  c.kernel = kp;
  b200::Engine e(nullptr, b200::to_abi(c), -1);
  b200::upload(e.h, set);
  double b[6];
  b200::bounds_to6(bounds, b);
  smcl_neighbor_stats st;
  b200::check(smcl_update_neighbors(e.h, pass_seed, b, &st));
  b200::download(e.h, set.neighbors.k_max, set);
  return b200::stats_from(st);
}

// solve_step(sys, lambda, limits) (gicp.cpp:47-75), fp64 on the device.
inline Tangent solve_step(const GnSystem& sys, double lambda, const StepLimits& limits = {}) {
  double H[36], b[6], out[6];
  for (int r = 0; r < 6; ++r) {
    b[r] = sys.b(r);
    for (int c = 0; c < 6; ++c) H[r * 6 + c] = sys.H(r, c);
  }
  b200::check(smcl_solve_step_batch(H, b, &lambda, 1, limits.omega_max, limits.v_max, out));
  Tangent t;
  for (int i = 0; i < 6; ++i) t(i) = out[i];
  return t;
}

// evaluate_all(map, nnf, scan, poses, params, steps, ll, nm) (gicp.cpp:87-107).
inline void evaluate_all(const GaussianCloud& map, const NearestNeighborField& nnf, const GaussianCloud& scan,
                         std::span<const Pose> poses, const GicpParams& params, std::span<Tangent> step_out,
                         std::span<double> log_lik_out, std::span<std::int32_t> n_matched_out) {
  if (step_out.size() != poses.size() || log_lik_out.size() != poses.size() || n_matched_out.size() != poses.size())
    throw std::invalid_argument("evaluate_all: output sizes must match poses");
  b200::Engine e(&map, b200::map_stage_config(nnf, params, static_cast<std::int64_t>(poses.size())), -1);
  b200::check_nnf(e.h, nnf);
  b200::upload_poses(e.h, poses);
  b200::CloudBuf s(scan, false);
  std::vector<double> steps(poses.size() * 6);
  b200::check(smcl_evaluate_all(e.h, &s.view, steps.data(), log_lik_out.data(), n_matched_out.data(), nullptr,
                                nullptr));
  for (std::size_t i = 0; i < poses.size(); ++i)
    for (int q = 0; q < 6; ++q) step_out[i](q) = steps[6 * i + q];
}

// evaluate_likelihoods(map, nnf, scan, poses, params, ll, nm) (gicp.cpp:109-137).
inline void evaluate_likelihoods(const GaussianCloud& map, const NearestNeighborField& nnf,
                                 const GaussianCloud& scan, std::span<const Pose> poses, const GicpParams& params,
                                 std::span<double> log_lik_out, std::span<std::int32_t> n_matched_out) {
  if (log_lik_out.size() != poses.size() || n_matched_out.size() != poses.size())
    throw std::invalid_argument("evaluate_likelihoods: output sizes must match poses");
  b200::Engine e(&map, b200::map_stage_config(nnf, params, static_cast<std::int64_t>(poses.size())), -1);
  b200::check_nnf(e.h, nnf);
  b200::upload_poses(e.h, poses);
  b200::CloudBuf s(scan, false);
  b200::check(smcl_evaluate_likelihoods(e.h, &s.view, log_lik_out.data(), n_matched_out.data()));
}

// compute_phis(poses, steps, idx, count, K, kp, phi) (svgd.cpp:36-49).
inline void compute_phis(std::span<const Pose> poses, std::span<const Tangent> steps,
                         std::span<const std::int32_t> neighbor_idx, std::span<const std::int32_t> neighbor_count,
                         int k_stride, const KernelParams& kp, std::span<Tangent> phi_out) {
  const std::size_t n = poses.size();
  if (steps.size() != n || phi_out.size() != n || neighbor_count.size() != n ||
      neighbor_idx.size() != n * static_cast<std::size_t>(k_stride))
    throw std::invalid_argument("compute_phis: size mismatch");
  FilterConfig c;
  c.n_particles = static_cast<int>(n);
  c.lsh.k_neighbors = k_stride;
  c.kernel = kp;
  b200::Engine e(nullptr, b200::to_abi(c), -1);
  ParticleSet s;
  s.poses.assign(poses.begin(), poses.end());
  s.neighbors.k_max = k_stride;
  s.neighbors.idx.assign(neighbor_idx.begin(), neighbor_idx.end());
  s.neighbors.kval.assign(neighbor_idx.size(), 0.0f);
  s.neighbors.count.assign(neighbor_count.begin(), neighbor_count.end());
  b200::upload(e.h, s);
  std::vector<double> st(n * 6), phi(n * 6);
  for (std::size_t i = 0; i < n; ++i)
    for (int q = 0; q < 6; ++q) st[6 * i + q] = steps[i](q);
  b200::check(smcl_compute_phis(e.h, st.data(), phi.data()));
  for (std::size_t i = 0; i < n; ++i)
    for (int q = 0; q < 6; ++q) phi_out[i](q) = phi[6 * i + q];
}

// apply_updates(poses, phis) (svgd.cpp:51-62).
inline void apply_updates(std::span<Pose> poses, std::span<const Tangent> phis) {
  if (phis.size() != poses.size()) throw std::invalid_argument("apply_updates: one phi per pose");
  FilterConfig c;
  c.n_particles = static_cast<int>(poses.size());
  c.lsh.k_neighbors = 1;
  b200::Engine e(nullptr, b200::to_abi(c), -1);
  b200::upload_poses(e.h, std::span<const Pose>(poses.data(), poses.size()));
  std::vector<double> ph(poses.size() * 6);
  for (std::size_t i = 0; i < poses.size(); ++i)
    for (int q = 0; q < 6; ++q) ph[6 * i + q] = phis[i](q);
  b200::check(smcl_apply_updates(e.h, ph.data()));
  ParticleSet s;
  b200::download(e.h, 1, s);
  for (std::size_t i = 0; i < poses.size(); ++i) poses[i] = s.poses[i];
}

namespace b200 {
// Posterior stages on a transient engine holding log_post (and the graph).
inline Engine* posterior_engine(std::span<const double> log_post, const NeighborGraph* g, std::unique_ptr<Engine>& own) {
  FilterConfig c;
  c.n_particles = static_cast<int>(log_post.size());
  c.lsh.k_neighbors = g ? g->k_max : 1;
  own = std::make_unique<Engine>(nullptr, to_abi(c), -1);
  ParticleSet s;
  s.poses.resize(log_post.size());
  s.log_post.assign(log_post.begin(), log_post.end());
  if (g) s.neighbors = *g;
  s.neighbors.k_max = c.lsh.k_neighbors;
  upload(own->h, s);
  return own.get();
}
inline void read_log_post(smcl_engine* h, int k, std::span<double> out) {
  ParticleSet s;
  download(h, k, s);
  std::memcpy(out.data(), s.log_post.data(), out.size() * sizeof(double));
}
}  // namespace b200

// normalize_log_post(log_post, floor) (posterior.cpp:13-24).
inline void normalize_log_post(std::span<double> log_post, double floor = k_default_log_post_floor) {
  std::unique_ptr<b200::Engine> own;
  b200::Engine* e = b200::posterior_engine(log_post, nullptr, own);
  b200::check(smcl_normalize_log_post(e->h, floor));
  b200::read_log_post(e->h, 1, log_post);
}

// bayes_update(log_post, ll, nm, beta, floor) (posterior.cpp:26-58): true when
// the observation was rejected (no particle matched; uniform reset).
inline bool bayes_update(std::span<double> log_post, std::span<const double> log_lik,
                         std::span<const std::int32_t> n_matched, double beta,
                         double floor = k_default_log_post_floor) {
  if (log_lik.size() != log_post.size() || n_matched.size() != log_post.size())
    throw std::invalid_argument("bayes_update: size mismatch");
  std::unique_ptr<b200::Engine> own;
  b200::Engine* e = b200::posterior_engine(log_post, nullptr, own);
  int32_t rejected = 0;
  b200::check(smcl_bayes_update(e->h, log_lik.data(), n_matched.data(), beta, floor, &rejected));
  b200::read_log_post(e->h, 1, log_post);
  return rejected != 0;
}

// smooth(log_post, graph, iters, floor) (posterior.cpp:60-97).
inline void smooth(std::span<double> log_post, const NeighborGraph& graph, int iters,
                   double floor = k_default_log_post_floor) {
  if (graph.size() != log_post.size()) throw std::invalid_argument("smooth: graph not initialized");
  std::unique_ptr<b200::Engine> own;
  b200::Engine* e = b200::posterior_engine(log_post, &graph, own);
  b200::check(smcl_smooth(e->h, iters, floor));
  b200::read_log_post(e->h, graph.k_max, log_post);
}

// representative(log_post, poses) (posterior.cpp:99-108).
inline Representative representative(std::span<const double> log_post, std::span<const Pose> poses) {
  Representative r;
  if (log_post.empty()) return r;
  if (poses.size() != log_post.size()) throw std::invalid_argument("representative: size mismatch");
  FilterConfig c;
  c.n_particles = static_cast<int>(poses.size());
  c.lsh.k_neighbors = 1;
  b200::Engine e(nullptr, b200::to_abi(c), -1);
  ParticleSet s;
  s.poses.assign(poses.begin(), poses.end());
  s.log_post.assign(log_post.begin(), log_post.end());
  s.neighbors.k_max = 1;
  b200::upload(e.h, s);
  double p[12];
  b200::check(smcl_representative(e.h, &r.index, p, &r.log_post));
  r.pose = b200::pose_from12(p);
  return r;
}

// ------------------------------------------------------------------ engine
// FilterEngine (filter.hpp:104-130 / filter.cpp:102-213) on one B200. The
// particle state lives in HBM; particles() downloads a host mirror lazily and
// mutable_particles() marks it for upload before the next step.
class FilterEngine {
 public:
  FilterEngine(GaussianCloud map, FilterConfig cfg) : map_(std::move(map)), cfg_(cfg) {
    if (map_.empty()) throw std::invalid_argument("FilterEngine: empty map");
    const smcl_config c = b200::to_abi(cfg_);
    b200::CloudBuf m(map_);
    b200::check(smcl_create(&m.view, &c, cfg_.device, &h_));
  }
  ~FilterEngine() {
    if (h_) smcl_destroy(h_);
  }
  FilterEngine(const FilterEngine&) = delete;
  FilterEngine& operator=(const FilterEngine&) = delete;

  void init_uniform(const Aabb& bounds) {
    double b[6];
    b200::bounds_to6(bounds, b);
    b200::check(smcl_init_uniform(h_, b));
    mirror_valid_ = dirty_ = false;
  }

  FrameResult step(const GaussianCloud& scan, const OdometryInput& odo) {
    flush();
    b200::CloudBuf s(scan, false);
    const smcl_odom o = b200::odom_from(odo);
    smcl_frame_result r;
    b200::check(smcl_step(h_, &s.view, &o, &r));
    mirror_valid_ = false;
    return b200::result_from(r);
  }

  // Raw sensor points: make_scan_cloud on the device, then step()
  // (the scenario runner's frame, scenario.cpp:315-338, in one call).
  FrameResult step_points(std::span<const Vec3> points, const OdometryInput& odo) {
    flush();
    std::vector<double> p(points.size() * 3);
    for (std::size_t i = 0; i < points.size(); ++i)
      for (int a = 0; a < 3; ++a) p[3 * i + a] = points[i](a);
    const smcl_odom o = b200::odom_from(odo);
    smcl_frame_result r;
    b200::check(smcl_step_points(h_, p.data(), static_cast<int64_t>(points.size()), &o, &r));
    mirror_valid_ = false;
    return b200::result_from(r);
  }

  const ParticleSet& particles() const {
    if (!mirror_valid_) download();
    return mirror_;
  }
  ParticleSet& mutable_particles() {
    if (!mirror_valid_) download();
    dirty_ = true;
    return mirror_;
  }
  const GaussianCloud& map() const { return map_; }
  const NearestNeighborField& nnf() const {
    if (nnf_.cells.empty()) {
      double origin[3], res = 0.0;
      b200::check(smcl_get_nnf(h_, nnf_.dims, origin, &res, nullptr));
      nnf_.cells.resize(static_cast<std::size_t>(nnf_.dims[0]) * nnf_.dims[1] * nnf_.dims[2]);
      b200::check(smcl_get_nnf(h_, nnf_.dims, origin, &res, nnf_.cells.data()));
      for (int a = 0; a < 3; ++a) nnf_.origin(a) = origin[a];
      nnf_.resolution = res;
      nnf_.max_query_dist = cfg_.nnf_max_query_dist;
      nnf_.padding = cfg_.nnf_padding;
    }
    return nnf_;
  }
  const FilterConfig& config() const { return cfg_; }
  std::int64_t frame_index() const { return smcl_frame_index(h_); }
  smcl_engine* handle() { return h_; }

 private:
  void download() const {
    b200::download(h_, cfg_.lsh.k_neighbors, mirror_);
    mirror_valid_ = true;
    dirty_ = false;
  }
  void flush() {
    if (!dirty_) return;
    b200::upload(h_, mirror_);
    dirty_ = false;
  }

  GaussianCloud map_;
  FilterConfig cfg_;
  smcl_engine* h_ = nullptr;
  mutable NearestNeighborField nnf_;
  mutable ParticleSet mirror_;
  mutable bool mirror_valid_ = false, dirty_ = false;
};

}  // namespace steinmcl
