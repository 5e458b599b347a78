// steinmcl_b200.hpp — header-only C++ facade over the C ABI (smcl_gpu.h) with
// the reference's names and call shapes (/root/reference/proj/include/steinmcl/
// filter.hpp:17-130, gaussian_cloud.hpp:21-40, posterior.hpp, neighbor_search.hpp).
//
// Differences a reference user has to know:
//  * No Eigen in the signatures: Pose stores R row-major in a double[9] and t
//    in a double[3]; define STEINMCL_B200_EIGEN before including this header
//    (after <Eigen/Core>) to get to_eigen/from_eigen converters.
//  * particles() returns a host mirror that is downloaded lazily;
//    mutable_particles() marks it dirty and it is uploaded before the next
//    device call (filter.hpp:111-113 semantics).
//  * Errors come back as the exception types the reference throws.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "smcl_gpu.h"

#ifdef STEINMCL_B200_EIGEN
#include <Eigen/Core>
#endif

namespace steinmcl_b200 {

struct Pose {  // se3.hpp:30-59 (R row-major)
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double t[3] = {0, 0, 0};
  static Pose identity() { return {}; }
};

struct Aabb {  // gaussian_cloud.hpp:21-31
  double min[3] = {0, 0, 0};
  double max[3] = {0, 0, 0};
};

struct GaussianCloud {  // gaussian_cloud.hpp:32-40: mu n*3, sigma n*9 row-major
  std::vector<double> mu, sigma;
  Aabb bounds;
  bool has_bounds = false;
  std::size_t size() const { return mu.size() / 3; }
  bool empty() const { return mu.empty(); }
};

struct OdometryInput {  // filter.hpp:56-60
  Pose delta;
  double cov[36] = {};
  bool valid = true;
};

using FilterConfig = smcl_config;  // filter.hpp:17-51 (flattened)
inline FilterConfig default_config() {
  FilterConfig c;
  smcl_config_default(&c);
  return c;
}

struct ParticleSet {  // particle_set.hpp:16-27 (+ NeighborGraph, neighbor_graph.hpp:16-22)
  std::vector<Pose> poses;
  std::vector<double> log_post;
  std::vector<std::int32_t> id;
  int k_max = 20;
  std::vector<std::int32_t> idx;
  std::vector<float> kval;
  std::vector<std::int32_t> count;
  std::size_t size() const { return poses.size(); }
};

using FrameResult = smcl_frame_result;  // filter.hpp:62-82

namespace detail {
inline void check(int rc) {
  if (rc == SMCL_OK) return;
  const std::string msg = smcl_last_error();
  if (rc == SMCL_EINVAL) throw std::invalid_argument(msg);
  if (rc == SMCL_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}
inline smcl_cloud view(const GaussianCloud& c, double* bounds_buf) {
  smcl_cloud v{static_cast<int64_t>(c.size()), c.mu.data(), c.sigma.data(), nullptr};
  if (c.has_bounds) {
    for (int a = 0; a < 3; ++a) {
      bounds_buf[a] = c.bounds.min[a];
      bounds_buf[3 + a] = c.bounds.max[a];
    }
    v.bounds = bounds_buf;
  }
  return v;
}
}  // namespace detail

// FilterEngine (filter.hpp:104-130) on one B200.
class FilterEngine {
 public:
  FilterEngine(const GaussianCloud& map, const FilterConfig& cfg, int device = 0) : cfg_(cfg) {
    double b[6];
    const smcl_cloud m = detail::view(map, b);
    detail::check(smcl_create(&m, &cfg_, device, &h_));
  }
  ~FilterEngine() {
    if (h_) smcl_destroy(h_);
  }
  FilterEngine(const FilterEngine&) = delete;
  FilterEngine& operator=(const FilterEngine&) = delete;

  void init_uniform(const Aabb& bounds) {
    const double b[6] = {bounds.min[0], bounds.min[1], bounds.min[2], bounds.max[0], bounds.max[1], bounds.max[2]};
    detail::check(smcl_init_uniform(h_, b));
    mirror_valid_ = dirty_ = false;
  }

  FrameResult step(const GaussianCloud& scan, const OdometryInput& odo) {
    flush();
    double b[6];
    const smcl_cloud s = detail::view(scan, b);
    smcl_odom o;
    std::memcpy(o.delta, odo.delta.R, sizeof(odo.delta.R));
    std::memcpy(o.delta + 9, odo.delta.t, sizeof(odo.delta.t));
    std::memcpy(o.cov, odo.cov, sizeof(o.cov));
    o.valid = odo.valid ? 1 : 0;
    FrameResult r;
    detail::check(smcl_step(h_, &s, &o, &r));
    mirror_valid_ = false;
    return r;
  }

  // Scenario-runner frame (scenario.cpp:315-338): make_scan_cloud on the
  // device from raw sensor points (x, y, z triples), then step().
  FrameResult step_points(const double* points_xyz, std::int64_t n_points, const OdometryInput& odo) {
    flush();
    smcl_odom o;
    std::memcpy(o.delta, odo.delta.R, sizeof(odo.delta.R));
    std::memcpy(o.delta + 9, odo.delta.t, sizeof(odo.delta.t));
    std::memcpy(o.cov, odo.cov, sizeof(o.cov));
    o.valid = odo.valid ? 1 : 0;
    FrameResult r;
    detail::check(smcl_step_points(h_, points_xyz, n_points, &o, &r));
    mirror_valid_ = false;
    return r;
  }

  const ParticleSet& particles() {
    if (!mirror_valid_) download();
    return mirror_;
  }
  ParticleSet& mutable_particles() {
    if (!mirror_valid_) download();
    dirty_ = true;
    return mirror_;
  }
  const FilterConfig& config() const { return cfg_; }
  std::int64_t frame_index() const { return smcl_frame_index(h_); }
  smcl_engine* handle() { return h_; }

 private:
  void download() {
    const std::int64_t n = smcl_num_particles(h_);
    mirror_.poses.resize(static_cast<std::size_t>(n));
    mirror_.log_post.resize(static_cast<std::size_t>(n));
    mirror_.id.resize(static_cast<std::size_t>(n));
    mirror_.k_max = cfg_.k_neighbors;
    mirror_.idx.resize(static_cast<std::size_t>(n) * cfg_.k_neighbors);
    mirror_.kval.resize(static_cast<std::size_t>(n) * cfg_.k_neighbors);
    mirror_.count.resize(static_cast<std::size_t>(n));
    std::vector<double> poses(static_cast<std::size_t>(n) * 12);
    smcl_particles_view v{n, cfg_.k_neighbors, poses.data(), mirror_.log_post.data(), mirror_.id.data(),
                          mirror_.idx.data(), mirror_.kval.data(), mirror_.count.data()};
    detail::check(smcl_get_particles(h_, &v));
    for (std::int64_t i = 0; i < n; ++i) {
      std::memcpy(mirror_.poses[static_cast<std::size_t>(i)].R, &poses[static_cast<std::size_t>(12 * i)], 72);
      std::memcpy(mirror_.poses[static_cast<std::size_t>(i)].t, &poses[static_cast<std::size_t>(12 * i + 9)], 24);
    }
    mirror_valid_ = true;
    dirty_ = false;
  }
  void flush() {
    if (!dirty_) return;
    const std::int64_t n = static_cast<std::int64_t>(mirror_.size());
    std::vector<double> poses(static_cast<std::size_t>(n) * 12);
    for (std::int64_t i = 0; i < n; ++i) {
      std::memcpy(&poses[static_cast<std::size_t>(12 * i)], mirror_.poses[static_cast<std::size_t>(i)].R, 72);
      std::memcpy(&poses[static_cast<std::size_t>(12 * i + 9)], mirror_.poses[static_cast<std::size_t>(i)].t, 24);
    }
    smcl_particles_view v{n, mirror_.k_max, poses.data(), mirror_.log_post.data(), mirror_.id.data(),
                          mirror_.idx.data(), mirror_.kval.data(), mirror_.count.data()};
    detail::check(smcl_set_particles(h_, &v));
    dirty_ = false;
  }

  FilterConfig cfg_;
  smcl_engine* h_ = nullptr;
  ParticleSet mirror_;
  bool mirror_valid_ = false, dirty_ = false;
};

// make_scan_cloud (filter.cpp:86-100) on the host.
inline GaussianCloud make_scan_cloud(const std::vector<double>& points_xyz, const FilterConfig& cfg) {
  const std::int64_t n = static_cast<std::int64_t>(points_xyz.size() / 3);
  GaussianCloud out;
  out.mu.resize(static_cast<std::size_t>(n) * 3);
  out.sigma.resize(static_cast<std::size_t>(n) * 9);
  std::int64_t m = 0;
  detail::check(smcl_make_scan_cloud(points_xyz.data(), n, &cfg, out.mu.data(), out.sigma.data(), &m));
  out.mu.resize(static_cast<std::size_t>(m) * 3);
  out.sigma.resize(static_cast<std::size_t>(m) * 9);
  return out;
}

#ifdef STEINMCL_B200_EIGEN
// Reference Pose (Eigen column-major Mat3 R, Vec3 t) <-> facade Pose.
template <class RefPose>
inline Pose from_eigen(const RefPose& p) {
  Pose q;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) q.R[r * 3 + c] = p.R(r, c);
    q.t[r] = p.t(r);
  }
  return q;
}
template <class RefPose>
inline RefPose to_eigen(const Pose& q) {
  RefPose p;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) p.R(r, c) = q.R[r * 3 + c];
    p.t(r) = q.t[r];
  }
  return p;
}
#endif

}  // namespace steinmcl_b200
