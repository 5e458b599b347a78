// Uses the reference-shaped C++ facade (include/steinmcl_b200.hpp) the way
// the reference's own callers use steinmcl::FilterEngine (scenario.cpp:315-338):
// build a map, init uniformly, step with scans and odometry, read the result.
// Exit code 0 and one line "facade_demo ok <rep_id> <total_ms>" on success.
#include <cstdio>
#include <vector>

#include "steinmcl_b200.hpp"

using namespace steinmcl_b200;

int main() {
  // Box room 8x6x3 m sampled at 60 points/m^2 (world.cpp:135-160).
  const double size[3] = {8.0, 6.0, 3.0};
  double rects[6 * 9];
  int32_t n_rects = 0;
  detail::check(smcl_sim_box_room(size, rects, 6, &n_rects));
  int64_t n_map = 0;
  detail::check(smcl_sim_sample_world(rects, n_rects, 60.0, 3, 10, 1e-3, nullptr, nullptr, &n_map));
  GaussianCloud map;
  map.mu.resize(static_cast<size_t>(n_map) * 3);
  map.sigma.resize(static_cast<size_t>(n_map) * 9);
  detail::check(smcl_sim_sample_world(rects, n_rects, 60.0, 3, 10, 1e-3, map.mu.data(), map.sigma.data(), &n_map));

  FilterConfig cfg = default_config();
  cfg.n_particles = 4096;
  cfg.nnf_resolution = 0.2;
  FilterEngine engine(map, cfg, 0);
  Aabb b;
  for (int a = 0; a < 3; ++a) b.max[a] = size[a];
  engine.init_uniform(b);

  smcl_sensor_spec sensor;
  smcl_sim_default_sensor(&sensor);
  Pose gt;
  gt.t[0] = 4.0;
  gt.t[1] = 3.0;
  gt.t[2] = 1.5;
  OdometryInput odo;
  odo.delta.t[0] = 0.05;
  for (int d = 0; d < 6; ++d) odo.cov[d * 7] = 1e-4;
  FrameResult r{};
  for (int f = 0; f < 3; ++f) {
    gt.t[0] += 0.05;
    double pose[12];
    for (int q = 0; q < 9; ++q) pose[q] = gt.R[q];
    for (int q = 0; q < 3; ++q) pose[9 + q] = gt.t[q];
    std::vector<double> pts(static_cast<size_t>(sensor.n_azimuth) * sensor.n_elevations * 3);
    uint64_t rng = 100 + static_cast<uint64_t>(f);
    int64_t n_pts = 0;
    detail::check(smcl_sim_scan(rects, n_rects, pose, &sensor, &rng, pts.data(), &n_pts));
    pts.resize(static_cast<size_t>(n_pts) * 3);
    // frames 0-1: host make_scan_cloud + step(); frame 2: raw points, scan
    // preparation on the device (step_points)
    r = f < 2 ? engine.step(make_scan_cloud(pts, cfg), odo) : engine.step_points(pts.data(), n_pts, odo);
  }
  const ParticleSet& ps = engine.particles();
  if (ps.size() != 4096) return 1;
  std::printf("facade_demo ok %d %.3f\n", r.rep_id, r.total_ms);
  return 0;
}
