// ORACLE — test infrastructure only (see omath.hpp header). Data model and
// hot-path function declarations restating /root/reference/proj/include/steinmcl/*.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "omath.hpp"

namespace orc {

// gaussian_cloud.hpp:21-40
struct Aabb {
  V3 min, max;
  V3 extent() const { return max - min; }
  bool contains(const V3& p) const {
    for (int a = 0; a < 3; ++a)
      if (!(p[a] >= min[a] && p[a] <= max[a])) return false;
    return true;
  }
  Aabb padded(double pad) const {
    return {v3(min[0] - pad, min[1] - pad, min[2] - pad), v3(max[0] + pad, max[1] + pad, max[2] + pad)};
  }
};

struct GaussianCloud {
  std::vector<V3> mu;
  std::vector<M3> sigma;
  Aabb bounds;
  std::size_t size() const { return mu.size(); }
  bool empty() const { return mu.empty(); }
};

Aabb compute_bounds(std::span<const V3> points);                                  // gaussian_cloud.cpp:14-22
GaussianCloud estimate_covariances(std::span<const V3> points, int k, double eps);  // gaussian_cloud.cpp:36-90
std::vector<V3> voxel_downsample(std::span<const V3> points, double leaf);         // gaussian_cloud.cpp:110-132
std::vector<V3> downsample_to(std::span<const V3> points, std::size_t max_points, double leaf0);  // 134-144
// Symmetric 3x3 eigen-decomposition, ascending eigenvalues; columns of V.
void sym_eig3(const M3& a, double w[3], M3& v);

// point_grid.hpp:15-46 / point_grid.cpp:10-141
class PointBucketGrid {
 public:
  PointBucketGrid(std::span<const V3> points, double cell_size);
  struct Neighbor {
    double dist2;
    std::int32_t index;
  };
  void k_nearest(const V3& query, int k, std::vector<Neighbor>& out) const;
  std::int32_t nearest_within(const V3& query, double max_dist) const;

 private:
  void cell_of(const V3& p, int c[3]) const;
  std::int32_t cell_index(int x, int y, int z) const { return (z * dims_[1] + y) * dims_[0] + x; }
  std::vector<V3> points_;
  std::vector<std::int32_t> order_, offsets_;
  V3 origin_;
  int dims_[3] = {0, 0, 0};
  double cell_size_ = 1.0;
};

// nnf.hpp:13-50
struct NearestNeighborField {
  static constexpr std::int32_t k_empty = -1;
  V3 origin;
  double resolution = 0.1;
  double max_query_dist = 1.0;
  int dims[3] = {0, 0, 0};
  std::vector<std::int32_t> cells;
  // nnf.hpp:24-35. Casts follow x86 cvttsd2si: out-of-int-range -> INT_MIN.
  std::int32_t lookup_nearest(const V3& p) const {
    const double inv = 1.0 / resolution;
    int c[3];
    for (int a = 0; a < 3; ++a) {
      const double f = std::floor((p[a] - origin[a]) * inv);
      c[a] = (f >= -2147483648.0 && f < 2147483648.0) ? static_cast<int>(f) : INT32_MIN;
    }
    if (static_cast<unsigned>(c[0]) >= static_cast<unsigned>(dims[0]) ||
        static_cast<unsigned>(c[1]) >= static_cast<unsigned>(dims[1]) ||
        static_cast<unsigned>(c[2]) >= static_cast<unsigned>(dims[2]))
      return k_empty;
    return cells[(static_cast<std::size_t>(c[2]) * dims[1] + c[1]) * dims[0] + c[0]];
  }
};
NearestNeighborField build_nnf(const GaussianCloud& map, double resolution, double padding,
                               double max_query_dist, std::size_t max_cells = std::size_t(1) << 30);

// ---------------------------------------------------------------- GICP (gicp.hpp)
inline constexpr double k_unmatched_log_lik = -1e30;
struct GnSystem {
  M6 H;
  V6 b;
  double log_lik = 0.0;
  int n_matched = 0;
};
struct GicpParams {
  double damping_scale = 1e-3;
  double omega_max = 0.5;
  double v_max = 1.0;
  double min_match_fraction = 0.5;
  double miss_cost = 25.0;
};
GnSystem evaluate(const GaussianCloud& map, const NearestNeighborField& nnf,
                  const GaussianCloud& scan, const Pose& pose);
V6 solve_step(const GnSystem& sys, double lambda, double omega_max, double v_max);
void evaluate_all(const GaussianCloud& map, const NearestNeighborField& nnf,
                  const GaussianCloud& scan, std::span<const Pose> poses, const GicpParams& p,
                  std::span<V6> step_out, std::span<double> ll_out, std::span<std::int32_t> nm_out,
                  GnSystem* sys_out = nullptr, bool serial = false);
void evaluate_likelihoods(const GaussianCloud& map, const NearestNeighborField& nnf,
                          const GaussianCloud& scan, std::span<const Pose> poses,
                          const GicpParams& p, std::span<double> ll_out,
                          std::span<std::int32_t> nm_out, bool serial = false);

// ---------------------------------------------------------------- SVGD (svgd.hpp)
struct KernelParams {
  double sigma_r = 5.0;
  double sigma_t = 2.5;
  double repulsion_gain = 1.0;
};
inline double kernel_of_tangent(const V6& d, const KernelParams& kp) {  // svgd.hpp:30-34
  const double qr = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
  const double qt = (d[3] * d[3] + d[4] * d[4]) + d[5] * d[5];
  return std::exp(-(kp.sigma_r * qr + kp.sigma_t * qt));
}
inline double kernel(const Pose& a, const Pose& b, const KernelParams& kp) {
  return kernel_of_tangent(se3_log(compose(inverse(a), b)), kp);
}
inline bool kernel_underflows(const Pose& a, const Pose& b, const KernelParams& kp) {  // svgd.hpp:45-47
  return kp.sigma_t * sqnorm(b.t - a.t) > 110.0;
}
V6 kernel_grad(const Pose& a, const Pose& b, const KernelParams& kp);  // svgd.hpp:53-60
V6 compute_phi(std::int32_t i, std::span<const Pose> poses, std::span<const V6> steps,
               std::span<const std::int32_t> nbrs, const KernelParams& kp);
void compute_phis(std::span<const Pose> poses, std::span<const V6> steps,
                  std::span<const std::int32_t> idx, std::span<const std::int32_t> count, int k_stride,
                  const KernelParams& kp, std::span<V6> phi_out, bool serial = false);
void apply_updates(std::span<Pose> poses, std::span<const V6> phis, bool serial = false);

// ---------------------------------------------------------------- graph / LSH
struct NeighborGraph {  // neighbor_graph.hpp:16-91
  int k_max = 20;
  std::vector<std::int32_t> idx;
  std::vector<float> kval;
  std::vector<std::int32_t> count;
  std::size_t size() const { return count.size(); }
  void init_self(std::size_t n, int k);
  void offer(std::size_t i, std::int32_t j, float k_ij);
  void refresh(std::size_t i, std::span<const Pose> poses, const KernelParams& kp);
};

struct ParticleSet {  // particle_set.hpp:16-27
  std::vector<Pose> poses;
  std::vector<double> log_post;
  std::vector<std::int32_t> id;
  NeighborGraph neighbors;
  std::size_t size() const { return poses.size(); }
  void reorder(std::span<const std::int32_t> old_of_new);
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
struct NeighborStats {
  std::int64_t n_buckets = 0, buckets_used = 0, overflow_dropped = 0;
  std::vector<std::int64_t> occupancy_hist;
  double mean_kernel = 0.0;
};
std::uint64_t lsh_hash(const Pose& pose, const Pose& frame, const V6& noise, const LshConfig& cfg,
                       const KernelParams& kp);
Pose random_lsh_frame(SplitMix64& rng, const Aabb& bounds);
std::int32_t next_prime_at_least(std::int32_t n);
NeighborStats update_neighbors(ParticleSet& set, const LshConfig& cfg, const KernelParams& kp,
                               std::uint64_t pass_seed, const Aabb& bounds);
NeighborStats update_neighbors_serial(ParticleSet& set, const LshConfig& cfg, const KernelParams& kp,
                                      std::uint64_t pass_seed, const Aabb& bounds);  // reference.cpp:78-167
std::vector<std::vector<std::int32_t>> brute_force_kernel_knn(std::span<const Pose> poses, int k,
                                                              const KernelParams& kp);

// ---------------------------------------------------------------- posterior
inline constexpr double k_default_log_post_floor = -80.0;
void normalize_log_post(std::span<double> log_post, double floor);
bool bayes_update(std::span<double> log_post, std::span<const double> ll,
                  std::span<const std::int32_t> nm, double beta, double floor);
void smooth(std::span<double> log_post, const NeighborGraph& g, int iters, double floor,
            bool serial = false);
ArgMax representative(std::span<const double> log_post);

// ---------------------------------------------------------------- filter (filter.hpp)
struct FilterConfig {
  int n_particles = 10000;
  KernelParams kernel;
  LshConfig lsh;
  double nnf_resolution = 0.1, nnf_max_query_dist = 1.0, nnf_padding = 0.5;
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
  double diffusion_sigma_rot = 0.02, diffusion_sigma_trans = 0.5;
  bool full_rotation = true;
  std::uint64_t seed = 1;
};
struct OdometryInput {
  Pose delta;
  M6 cov;
  bool valid = true;
};
struct FrameResult {
  Pose representative;
  double rep_log_post = 0.0;
  std::int64_t rep_index = -1;
  std::int32_t rep_id = -1;
  std::size_t n_particles = 0;
  double mean_n_matched = 0.0;
  bool scan_empty = false, observation_rejected = false;
  NeighborStats neighbor_stats;
  double times_ms[6] = {0, 0, 0, 0, 0, 0};  // predict, neighbor, likelihood, update, posterior, total
};

M6 covariance_sqrt(const M6& cov);  // filter.cpp:25-35
ParticleSet init_uniform(const FilterConfig& cfg, const Aabb& bounds, bool full_rotation,
                         std::uint64_t seed);
void predict(ParticleSet& set, const Pose& delta, const M6& cov, std::uint64_t frame_seed);
GaussianCloud make_scan_cloud(std::span<const V3> points, const FilterConfig& cfg);

class FilterEngine {  // filter.hpp:104-130
 public:
  FilterEngine(GaussianCloud map, FilterConfig cfg);
  void init_uniform(const Aabb& bounds);
  FrameResult step(const GaussianCloud& scan, const OdometryInput& odo);
  ParticleSet& particles() { return particles_; }
  const NearestNeighborField& nnf() const { return nnf_; }
  const GaussianCloud& map() const { return map_; }
  std::int64_t frame_index() const { return frame_; }
  // Test harness only (no reference counterpart): start an oracle engine at
  // another engine's frame index, so both derive the same per-frame seeds.
  void set_frame_index(std::int64_t f) { frame_ = f; }
  const FilterConfig& config() const { return cfg_; }

 private:
  GaussianCloud map_;
  FilterConfig cfg_;
  NearestNeighborField nnf_;
  ParticleSet particles_;
  std::int64_t frame_ = 0;
  std::vector<V6> steps_, phis_;
  std::vector<double> log_lik_;
  std::vector<std::int32_t> n_matched_;
};

}  // namespace orc
