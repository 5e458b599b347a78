// A reference-shaped call site compiled against the source-compatible facade
// (include/steinmcl/*.hpp -> steinmcl/b200.hpp). Part 1 is written the way
// the reference's scenario runner drives the engine
// (/root/reference/proj/src/sim/scenario.cpp:315-338): FilterEngine(map, cfg),
// init_uniform(engine.map().bounds), step(scan, odo) per frame, reading
// fr.representative.t.x(), fr.times.*, fr.neighbor_stats. Part 2 composes the
// free stage functions exactly as FilterEngine::step does
// (/root/reference/proj/src/filter.cpp:118-213) and checks that they
// reproduce the engine's step bit for bit.
// Prints "scenario_callsite ok ..." and exits 0 on success.
#include <cstdio>
#include <cstring>
#include <vector>

#include "steinmcl/filter.hpp"
#include "steinmcl/rng.hpp"

using namespace steinmcl;

namespace {

// Synthetic inputs through the library's simulator entry points (a stand-in
// for the reference's sim/world.cpp, which is outside the filter API).
struct Room {
  std::vector<double> rects = std::vector<double>(6 * 9);
  int32_t n_rects = 0;
};

Room box_room(double sx, double sy, double sz) {
  Room r;
  const double size[3] = {sx, sy, sz};
  b200::check(smcl_sim_box_room(size, r.rects.data(), 6, &r.n_rects));
  return r;
}

GaussianCloud sample_world(const Room& w, double density, std::uint64_t seed, int k, double eps) {
  int64_t n = 0;
  b200::check(smcl_sim_sample_world(w.rects.data(), w.n_rects, density, seed, k, eps, nullptr, nullptr, &n));
  std::vector<double> mu(static_cast<size_t>(n) * 3), sigma(static_cast<size_t>(n) * 9);
  b200::check(smcl_sim_sample_world(w.rects.data(), w.n_rects, density, seed, k, eps, mu.data(), sigma.data(), &n));
  return b200::cloud_from(mu, sigma, n);
}

std::vector<Vec3> simulate_scan(const Room& w, const Pose& sensor_pose, std::uint64_t seed) {
  smcl_sensor_spec spec;
  smcl_sim_default_sensor(&spec);
  spec.n_azimuth = 128;
  double p[12];
  b200::pose_to12(sensor_pose, p);
  std::vector<double> pts(static_cast<size_t>(spec.n_azimuth) * spec.n_elevations * 3);
  int64_t n = 0;
  std::uint64_t rng = seed;
  b200::check(smcl_sim_scan(w.rects.data(), w.n_rects, p, &spec, &rng, pts.data(), &n));
  std::vector<Vec3> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[static_cast<size_t>(i)] = Vec3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  return out;
}

bool same(const ParticleSet& a, const ParticleSet& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    if (std::memcmp(&a.poses[i], &b.poses[i], sizeof(Pose)) != 0) return false;
    if (std::memcmp(&a.log_post[i], &b.log_post[i], sizeof(double)) != 0 || a.id[i] != b.id[i]) return false;
  }
  return a.neighbors.idx == b.neighbors.idx && a.neighbors.count == b.neighbors.count &&
         std::memcmp(a.neighbors.kval.data(), b.neighbors.kval.data(), a.neighbors.kval.size() * sizeof(float)) == 0;
}

}  // namespace

int main() {
  FilterConfig cfg;
  cfg.n_particles = 8192;
  cfg.nnf_resolution = 0.2;
  cfg.kernel.sigma_r = 5.0;
  cfg.lsh.k_neighbors = 20;
  cfg.gicp.miss_cost = 25.0;
  cfg.n_scan_max = 256;
  const Room world = box_room(8.0, 6.0, 3.0);
  const GaussianCloud map = sample_world(world, 60.0, mix_seed(cfg.seed, 7), cfg.covariance_k, cfg.epsilon_plane);

  // ---- Part 1: scenario.cpp:315-338 shape
  FilterEngine engine(map, cfg);
  engine.init_uniform(engine.map().bounds);
  Pose truth = Pose::identity();
  truth.t = Vec3(4.0, 3.0, 1.5);
  OdometryInput odo;
  odo.delta.t = Vec3(0.05, 0.0, 0.0);
  for (int d = 0; d < 6; ++d) odo.cov(d, d) = 1e-4;
  StageTimes sum_times;
  std::vector<Pose> estimated;
  FrameResult fr;
  for (int f = 0; f < 4; ++f) {
    truth = truth * odo.delta;
    const GaussianCloud scan = make_scan_cloud(simulate_scan(world, truth, 100 + f), cfg);
    fr = engine.step(scan, odo);
    estimated.push_back(fr.representative);
    sum_times.predict_ms += fr.times.predict_ms;
    sum_times.neighbor_ms += fr.times.neighbor_ms;
    sum_times.likelihood_ms += fr.times.likelihood_ms;
    sum_times.update_ms += fr.times.update_ms;
    sum_times.posterior_ms += fr.times.posterior_ms;
    sum_times.total_ms += fr.times.total_ms;
  }
  if (engine.frame_index() != 4 || engine.particles().size() != static_cast<size_t>(cfg.n_particles) ||
      fr.n_particles != static_cast<size_t>(cfg.n_particles) || fr.neighbor_stats.n_buckets <= 0 ||
      engine.nnf().lookup_nearest(Vec3(0.3, 3.0, 1.5)) == NearestNeighborField::k_empty ||
      engine.nnf().lookup_nearest(Vec3(4.0, 3.0, 1.5)) != NearestNeighborField::k_empty) {
    std::printf("scenario_callsite FAIL part 1\n");
    return 1;
  }

  // ---- Part 2: FilterEngine::step composed from the free stage functions
  FilterEngine e2(map, cfg);
  e2.init_uniform(e2.map().bounds);
  ParticleSet set = e2.particles();
  const GaussianCloud scan = make_scan_cloud(simulate_scan(world, truth, 200), cfg);
  const std::uint64_t frame = static_cast<std::uint64_t>(e2.frame_index());
  predict(set, odo.delta, odo.cov, mix_seed(cfg.seed, 2, frame));
  const NeighborStats nst = update_neighbors(set, cfg.lsh, cfg.kernel, mix_seed(cfg.seed, 3, frame), map.bounds);
  const size_t n = set.size();
  std::vector<Tangent> steps(n), phis(n);
  std::vector<double> ll(n);
  std::vector<std::int32_t> nm(n);
  evaluate_all(map, e2.nnf(), scan, set.poses, cfg.gicp, steps, ll, nm);
  compute_phis(set.poses, steps, set.neighbors.idx, set.neighbors.count, set.neighbors.k_max, cfg.kernel, phis);
  apply_updates(set.poses, phis);
  evaluate_likelihoods(map, e2.nnf(), scan, set.poses, cfg.gicp, ll, nm);
  const bool rejected = bayes_update(set.log_post, ll, nm, cfg.beta, cfg.log_post_floor);
  smooth(set.log_post, set.neighbors, cfg.smooth_iters, cfg.log_post_floor);
  const Representative rep = representative(set.log_post, set.poses);

  const FrameResult r2 = e2.step(scan, odo);
  const bool ok = same(set, e2.particles()) && rep.index == r2.rep_index && rep.log_post == r2.rep_log_post &&
                  rejected == r2.observation_rejected && nst.buckets_used == r2.neighbor_stats.buckets_used &&
                  set.id[static_cast<size_t>(rep.index)] == r2.rep_id;
  if (!ok) {
    std::printf("scenario_callsite FAIL part 2 (rep %lld vs %lld, log_post %.17g vs %.17g)\n",
                static_cast<long long>(rep.index), static_cast<long long>(r2.rep_index), rep.log_post,
                r2.rep_log_post);
    return 1;
  }
  std::printf("scenario_callsite ok frames=%zu rep=(%.3f %.3f %.3f) total_ms=%.3f stages_bitwise=1\n",
              estimated.size(), fr.representative.t.x(), fr.representative.t.y(), fr.representative.t.z(),
              sum_times.total_ms);
  return 0;
}
