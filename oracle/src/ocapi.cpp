// ORACLE — test infrastructure only. extern "C" surface of the CPU restatement,
// loaded by tests/ (ctypes) and by bench.py's cpu_baseline / --impl reference
// legs. It consumes the product's public ABI structs (include/smcl_gpu.h, plain
// C types) so both sides receive byte-identical inputs.
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "../../include/smcl_gpu.h"
#include "oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SMCL_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return SMCL_EINVAL;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return SMCL_ELOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SMCL_ERUNTIME;
  }
}

Pose load_pose(const double* p) {
  Pose q;
  for (int i = 0; i < 9; ++i) q.R.m[i] = p[i];
  for (int i = 0; i < 3; ++i) q.t[i] = p[9 + i];
  return q;
}
void store_pose(const Pose& q, double* p) {
  for (int i = 0; i < 9; ++i) p[i] = q.R.m[i];
  for (int i = 0; i < 3; ++i) p[9 + i] = q.t[i];
}
V6 load6(const double* x) {
  V6 v;
  for (int i = 0; i < 6; ++i) v[i] = x[i];
  return v;
}
Aabb load_bounds(const double* b) { return {v3(b[0], b[1], b[2]), v3(b[3], b[4], b[5])}; }
std::vector<V3> load_points(const double* p, std::int64_t n) {
  std::vector<V3> v(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) v[static_cast<std::size_t>(i)] = v3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
  return v;
}
GaussianCloud load_cloud(const smcl_cloud* c) {
  GaussianCloud g;
  if (!c || c->n == 0) return g;
  g.mu = load_points(c->mu, c->n);
  g.sigma.resize(static_cast<std::size_t>(c->n));
  for (std::int64_t i = 0; i < c->n; ++i)
    for (int k = 0; k < 9; ++k) g.sigma[static_cast<std::size_t>(i)].m[k] = c->sigma[9 * i + k];
  g.bounds = c->bounds ? load_bounds(c->bounds) : compute_bounds(g.mu);
  return g;
}
FilterConfig load_cfg(const smcl_config* c) {
  FilterConfig f;
  f.n_particles = c->n_particles;
  f.kernel = {c->sigma_r, c->sigma_t, c->repulsion_gain};
  f.lsh.alpha = c->lsh_alpha;
  f.lsh.noise_sigma = c->lsh_noise_sigma;
  f.lsh.buckets_factor = c->lsh_buckets_factor;
  f.lsh.n_buckets = c->lsh_n_buckets;
  f.lsh.bucket_capacity = c->lsh_bucket_capacity;
  f.lsh.k_neighbors = c->k_neighbors;
  f.lsh.reorder_particles = c->reorder_particles != 0;
  f.nnf_resolution = c->nnf_resolution;
  f.nnf_max_query_dist = c->nnf_max_query_dist;
  f.nnf_padding = c->nnf_padding;
  f.smooth_iters = c->smooth_iters;
  f.beta = c->beta;
  f.n_svgd_iters = c->n_svgd_iters;
  f.gn_scan_stride = c->gn_scan_stride;
  f.gicp = {c->damping_scale, c->omega_max, c->v_max, c->min_match_fraction, c->miss_cost};
  f.log_post_floor = c->log_post_floor;
  f.covariance_k = c->covariance_k;
  f.epsilon_plane = c->epsilon_plane;
  f.n_scan_max = c->n_scan_max;
  f.scan_voxel_leaf = c->scan_voxel_leaf;
  f.sensor_noise_sigma = c->sensor_noise_sigma;
  f.diffusion_sigma_rot = c->diffusion_sigma_rot;
  f.diffusion_sigma_trans = c->diffusion_sigma_trans;
  f.full_rotation = c->full_rotation != 0;
  f.seed = c->seed;
  return f;
}
LshConfig lsh_of(const smcl_config* c) { return load_cfg(c).lsh; }
KernelParams kp_of(const smcl_config* c) { return load_cfg(c).kernel; }

ParticleSet load_set(const smcl_particles_view* v) {
  ParticleSet s;
  const std::size_t n = static_cast<std::size_t>(v->n), k = static_cast<std::size_t>(v->k);
  s.poses.resize(n);
  for (std::size_t i = 0; i < n; ++i) s.poses[i] = load_pose(v->poses + 12 * i);
  s.log_post.assign(v->log_post, v->log_post + n);
  s.id.assign(v->id, v->id + n);
  s.neighbors.k_max = v->k;
  s.neighbors.idx.assign(v->idx, v->idx + n * k);
  s.neighbors.kval.assign(v->kval, v->kval + n * k);
  s.neighbors.count.assign(v->count, v->count + n);
  return s;
}
void store_set(const ParticleSet& s, smcl_particles_view* v) {
  const std::size_t n = s.size(), k = static_cast<std::size_t>(s.neighbors.k_max);
  v->n = static_cast<std::int64_t>(n);
  v->k = s.neighbors.k_max;
  for (std::size_t i = 0; i < n; ++i) store_pose(s.poses[i], v->poses + 12 * i);
  std::memcpy(v->log_post, s.log_post.data(), n * sizeof(double));
  std::memcpy(v->id, s.id.data(), n * sizeof(std::int32_t));
  std::memcpy(v->idx, s.neighbors.idx.data(), n * k * sizeof(std::int32_t));
  std::memcpy(v->kval, s.neighbors.kval.data(), n * k * sizeof(float));
  std::memcpy(v->count, s.neighbors.count.data(), n * sizeof(std::int32_t));
}
void store_stats(const NeighborStats& st, smcl_neighbor_stats* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  out->n_buckets = st.n_buckets;
  out->buckets_used = st.buckets_used;
  out->overflow_dropped = st.overflow_dropped;
  out->mean_kernel = st.mean_kernel;
  out->hist_len = static_cast<std::int32_t>(std::min<std::size_t>(st.occupancy_hist.size(), SMCL_MAX_HIST));
  for (int i = 0; i < out->hist_len; ++i) out->occupancy_hist[i] = st.occupancy_hist[static_cast<std::size_t>(i)];
}

struct OracleMap {
  GaussianCloud map;
  NearestNeighborField nnf;
};
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- primitives
void orc_se3_exp(const double* xi, double* pose) { store_pose(se3_exp(load6(xi)), pose); }
void orc_se3_log(const double* pose, double* xi) {
  const V6 v = se3_log(load_pose(pose));
  for (int i = 0; i < 6; ++i) xi[i] = v[i];
}
void orc_compose(const double* a, const double* b, double* out) { store_pose(compose(load_pose(a), load_pose(b)), out); }
void orc_inverse(const double* a, double* out) { store_pose(inverse(load_pose(a)), out); }
void orc_renormalize(double* pose) {
  Pose p = load_pose(pose);
  renormalize_if_needed(p);
  store_pose(p, pose);
}
double orc_rotation_drift(const double* pose) { return rotation_drift(load_pose(pose)); }
std::uint64_t orc_mix_seed(std::uint64_t a, std::uint64_t b) { return mix_seed(a, b); }
std::uint64_t orc_splitmix_next(std::uint64_t* state) {
  SplitMix64 g(*state);
  const std::uint64_t v = g();
  *state = g.state;
  return v;
}
void orc_normal6(std::uint64_t* state, double* z) {
  SplitMix64 g(*state);
  const V6 v = normal6(g);
  *state = g.state;
  for (int i = 0; i < 6; ++i) z[i] = v[i];
}
double orc_uniform01(std::uint64_t* state) {
  SplitMix64 g(*state);
  const double u = uniform01(g);
  *state = g.state;
  return u;
}
void orc_random_rotation(std::uint64_t* state, double* R) {
  SplitMix64 g(*state);
  const M3 r = random_rotation(g);
  *state = g.state;
  std::memcpy(R, r.m, 9 * sizeof(double));
}
double orc_kernel(const double* a, const double* b, double sr, double st) {
  return kernel(load_pose(a), load_pose(b), {sr, st, 1.0});
}
void orc_kernel_grad(const double* a, const double* b, double sr, double st, double* g) {
  const V6 v = kernel_grad(load_pose(a), load_pose(b), {sr, st, 1.0});
  for (int i = 0; i < 6; ++i) g[i] = v[i];
}
std::uint64_t orc_lsh_hash(const double* pose, const double* frame, const double* noise, double alpha, double sr,
                           double st) {
  LshConfig cfg;
  cfg.alpha = alpha;
  return lsh_hash(load_pose(pose), load_pose(frame), load6(noise), cfg, {sr, st, 1.0});
}
void orc_random_lsh_frame(std::uint64_t* state, const double* bounds, double* frame) {
  SplitMix64 g(*state);
  const Pose f = random_lsh_frame(g, load_bounds(bounds));
  *state = g.state;
  store_pose(f, frame);
}
std::int32_t orc_next_prime(std::int32_t n) { return next_prime_at_least(n); }
int orc_solve_step(const double* H, const double* b, double lambda, double omax, double vmax, double* out) {
  return guard([&] {
    GnSystem s;
    std::memcpy(s.H.m, H, 36 * sizeof(double));
    for (int i = 0; i < 6; ++i) s.b[i] = b[i];
    const V6 v = solve_step(s, lambda, omax, vmax);
    for (int i = 0; i < 6; ++i) out[i] = v[i];
  });
}
// solve_step over n systems (H row-major 36, b 6, lambda per system).
int orc_solve_step_batch(const double* H, const double* b, const double* lambda, std::int64_t n, double omax,
                         double vmax, double* out) {
  return guard([&] {
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < n; ++i) {
      GnSystem s;
      std::memcpy(s.H.m, H + 36 * i, 36 * sizeof(double));
      for (int q = 0; q < 6; ++q) s.b[q] = b[6 * i + q];
      const V6 v = solve_step(s, lambda[i], omax, vmax);
      for (int q = 0; q < 6; ++q) out[6 * i + q] = v[q];
    }
  });
}
void orc_covariance_sqrt(const double* cov, double* L) {
  M6 c;
  std::memcpy(c.m, cov, 36 * sizeof(double));
  const M6 l = covariance_sqrt(c);
  std::memcpy(L, l.m, 36 * sizeof(double));
}

// ---------------------------------------------------------------- map / scan prep
void* orc_map_create(const smcl_cloud* map, double res, double pad, double mqd) {
  void* out = nullptr;
  const int rc = guard([&] {
    auto m = std::make_unique<OracleMap>();
    m->map = load_cloud(map);
    m->nnf = build_nnf(m->map, res, pad, mqd);
    out = m.release();
  });
  return rc == SMCL_OK ? out : nullptr;
}
void orc_map_destroy(void* h) { delete static_cast<OracleMap*>(h); }
void orc_map_nnf(void* h, std::int32_t* dims, double* origin, std::int32_t* cells) {
  const auto* m = static_cast<OracleMap*>(h);
  for (int a = 0; a < 3; ++a) {
    dims[a] = m->nnf.dims[a];
    origin[a] = m->nnf.origin[a];
  }
  if (cells) std::memcpy(cells, m->nnf.cells.data(), m->nnf.cells.size() * sizeof(std::int32_t));
}
std::int32_t orc_map_lookup(void* h, const double* p) {
  return static_cast<OracleMap*>(h)->nnf.lookup_nearest(v3(p[0], p[1], p[2]));
}
int orc_estimate_covariances(const double* pts, std::int64_t n, int k, double eps, double* sigma_out) {
  return guard([&] {
    const auto v = load_points(pts, n);
    const GaussianCloud c = estimate_covariances(v, k, eps);
    for (std::size_t i = 0; i < c.size(); ++i) std::memcpy(sigma_out + 9 * i, c.sigma[i].m, 9 * sizeof(double));
  });
}
int orc_downsample_to(const double* pts, std::int64_t n, std::int64_t max_points, double leaf, double* out,
                      std::int64_t* n_out) {
  return guard([&] {
    const auto v = downsample_to(load_points(pts, n), static_cast<std::size_t>(max_points), leaf);
    for (std::size_t i = 0; i < v.size(); ++i)
      for (int a = 0; a < 3; ++a) out[3 * i + static_cast<std::size_t>(a)] = v[i][a];
    *n_out = static_cast<std::int64_t>(v.size());
  });
}
int orc_make_scan_cloud(const double* pts, std::int64_t n, const smcl_config* cfg, double* mu_out,
                        double* sigma_out, std::int64_t* n_out) {
  return guard([&] {
    const GaussianCloud c = make_scan_cloud(load_points(pts, n), load_cfg(cfg));
    for (std::size_t i = 0; i < c.size(); ++i) {
      for (int a = 0; a < 3; ++a) mu_out[3 * i + static_cast<std::size_t>(a)] = c.mu[i][a];
      std::memcpy(sigma_out + 9 * i, c.sigma[i].m, 9 * sizeof(double));
    }
    *n_out = static_cast<std::int64_t>(c.size());
  });
}

// ---------------------------------------------------------------- GICP
int orc_evaluate_all(void* maph, const smcl_cloud* scan, const double* poses, std::int64_t n, const smcl_config* cfg,
                     double* steps, double* ll, std::int32_t* nm, double* H, double* b, int serial) {
  return guard([&] {
    const auto* m = static_cast<OracleMap*>(maph);
    const GaussianCloud sc = load_cloud(scan);
    std::vector<Pose> ps(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) ps[static_cast<std::size_t>(i)] = load_pose(poses + 12 * i);
    std::vector<V6> st(ps.size());
    std::vector<GnSystem> sys(ps.size());
    std::vector<double> llv(ps.size());
    std::vector<std::int32_t> nmv(ps.size());
    evaluate_all(m->map, m->nnf, sc, ps, load_cfg(cfg).gicp, st, llv, nmv, sys.data(), serial != 0);
    for (std::size_t i = 0; i < ps.size(); ++i) {
      if (steps)
        for (int c = 0; c < 6; ++c) steps[6 * i + static_cast<std::size_t>(c)] = st[i][c];
      if (ll) ll[i] = llv[i];
      if (nm) nm[i] = nmv[i];
      if (H) std::memcpy(H + 36 * i, sys[i].H.m, 36 * sizeof(double));
      if (b)
        for (int c = 0; c < 6; ++c) b[6 * i + static_cast<std::size_t>(c)] = sys[i].b[c];
    }
  });
}
int orc_evaluate_likelihoods(void* maph, const smcl_cloud* scan, const double* poses, std::int64_t n,
                             const smcl_config* cfg, double* ll, std::int32_t* nm, int serial) {
  return guard([&] {
    const auto* m = static_cast<OracleMap*>(maph);
    const GaussianCloud sc = load_cloud(scan);
    std::vector<Pose> ps(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) ps[static_cast<std::size_t>(i)] = load_pose(poses + 12 * i);
    evaluate_likelihoods(m->map, m->nnf, sc, ps, load_cfg(cfg).gicp, std::span<double>(ll, ps.size()),
                         std::span<std::int32_t>(nm, ps.size()), serial != 0);
  });
}

// ---------------------------------------------------------------- particles
int orc_update_neighbors(smcl_particles_view* view, const smcl_config* cfg, std::uint64_t pass_seed,
                         const double* bounds, smcl_neighbor_stats* stats, int serial) {
  return guard([&] {
    ParticleSet s = load_set(view);
    const NeighborStats st = serial ? update_neighbors_serial(s, lsh_of(cfg), kp_of(cfg), pass_seed, load_bounds(bounds))
                                    : update_neighbors(s, lsh_of(cfg), kp_of(cfg), pass_seed, load_bounds(bounds));
    store_set(s, view);
    store_stats(st, stats);
  });
}
// NeighborGraph::init_self(1, k) followed by offer(0, js[q], kvs[q]) for each
// q (neighbor_graph.hpp:24-72); the final list of particle 0.
int orc_graph_offers(int k, const std::int32_t* js, const float* kvs, int n_offers, std::int32_t* idx_out,
                     float* kval_out, std::int32_t* count_out) {
  return guard([&] {
    NeighborGraph g;
    g.init_self(1, k);
    for (int q = 0; q < n_offers; ++q) g.offer(0, js[q], kvs[q]);
    for (int s = 0; s < k; ++s) {
      idx_out[s] = g.idx[static_cast<std::size_t>(s)];
      kval_out[s] = g.kval[static_cast<std::size_t>(s)];
    }
    *count_out = g.count[0];
  });
}
int orc_brute_knn(const double* poses, std::int64_t n, int k, double sr, double st, std::int32_t* out) {
  return guard([&] {
    std::vector<Pose> ps(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) ps[static_cast<std::size_t>(i)] = load_pose(poses + 12 * i);
    const auto lists = brute_force_kernel_knn(ps, k, {sr, st, 1.0});
    for (std::size_t i = 0; i < lists.size(); ++i)
      for (std::size_t s = 0; s < lists[i].size(); ++s) out[i * static_cast<std::size_t>(k) + s] = lists[i][s];
  });
}
int orc_compute_phis(const double* poses, const double* steps, const std::int32_t* idx, const std::int32_t* count,
                     std::int64_t n, int k, const smcl_config* cfg, double* phi_out, int serial) {
  return guard([&] {
    std::vector<Pose> ps(static_cast<std::size_t>(n));
    std::vector<V6> st(static_cast<std::size_t>(n)), phi(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) {
      ps[static_cast<std::size_t>(i)] = load_pose(poses + 12 * i);
      st[static_cast<std::size_t>(i)] = load6(steps + 6 * i);
    }
    compute_phis(ps, st, std::span<const std::int32_t>(idx, static_cast<std::size_t>(n * k)),
                 std::span<const std::int32_t>(count, static_cast<std::size_t>(n)), k, kp_of(cfg), phi, serial != 0);
    for (std::int64_t i = 0; i < n; ++i)
      for (int c = 0; c < 6; ++c) phi_out[6 * i + c] = phi[static_cast<std::size_t>(i)][c];
  });
}
int orc_apply_updates(double* poses, const double* phis, std::int64_t n) {
  return guard([&] {
    std::vector<Pose> ps(static_cast<std::size_t>(n));
    std::vector<V6> ph(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) {
      ps[static_cast<std::size_t>(i)] = load_pose(poses + 12 * i);
      ph[static_cast<std::size_t>(i)] = load6(phis + 6 * i);
    }
    apply_updates(ps, ph);
    for (std::int64_t i = 0; i < n; ++i) store_pose(ps[static_cast<std::size_t>(i)], poses + 12 * i);
  });
}
int orc_predict(double* poses, std::int64_t n, const double* delta, const double* cov, std::uint64_t frame_seed) {
  return guard([&] {
    ParticleSet s;
    s.poses.resize(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) s.poses[static_cast<std::size_t>(i)] = load_pose(poses + 12 * i);
    M6 c;
    std::memcpy(c.m, cov, 36 * sizeof(double));
    predict(s, load_pose(delta), c, frame_seed);
    for (std::int64_t i = 0; i < n; ++i) store_pose(s.poses[static_cast<std::size_t>(i)], poses + 12 * i);
  });
}
int orc_init_uniform(std::int64_t n, int k, const double* bounds, int full_rotation, std::uint64_t seed,
                     smcl_particles_view* out) {
  return guard([&] {
    FilterConfig cfg;
    cfg.n_particles = static_cast<int>(n);
    cfg.lsh.k_neighbors = k;
    const ParticleSet s = init_uniform(cfg, load_bounds(bounds), full_rotation != 0, seed);
    store_set(s, out);
  });
}

// ---------------------------------------------------------------- posterior
int orc_normalize_log_post(double* lp, std::int64_t n, double floor) {
  return guard([&] { normalize_log_post(std::span<double>(lp, static_cast<std::size_t>(n)), floor); });
}
int orc_bayes_update(double* lp, const double* ll, const std::int32_t* nm, std::int64_t n, double beta, double floor,
                     std::int32_t* rejected) {
  return guard([&] {
    const std::size_t u = static_cast<std::size_t>(n);
    *rejected = bayes_update(std::span<double>(lp, u), std::span<const double>(ll, u),
                             std::span<const std::int32_t>(nm, u), beta, floor);
  });
}
int orc_smooth(double* lp, const std::int32_t* idx, const float* kval, const std::int32_t* count, std::int64_t n, int k,
               int iters, double floor, int serial) {
  return guard([&] {
    NeighborGraph g;
    const std::size_t u = static_cast<std::size_t>(n), uk = u * static_cast<std::size_t>(k);
    g.k_max = k;
    g.idx.assign(idx, idx + uk);
    g.kval.assign(kval, kval + uk);
    g.count.assign(count, count + u);
    smooth(std::span<double>(lp, u), g, iters, floor, serial != 0);
  });
}
int orc_representative(const double* lp, std::int64_t n, std::int64_t* index, double* value) {
  return guard([&] {
    const ArgMax a = representative(std::span<const double>(lp, static_cast<std::size_t>(n)));
    *index = a.index;
    *value = a.value;
  });
}

// ---------------------------------------------------------------- engine
void* orc_engine_create(const smcl_cloud* map, const smcl_config* cfg) {
  void* out = nullptr;
  const int rc = guard([&] { out = new FilterEngine(load_cloud(map), load_cfg(cfg)); });
  return rc == SMCL_OK ? out : nullptr;
}
void orc_engine_destroy(void* h) { delete static_cast<FilterEngine*>(h); }
int orc_engine_init_uniform(void* h, const double* bounds) {
  return guard([&] { static_cast<FilterEngine*>(h)->init_uniform(load_bounds(bounds)); });
}
int orc_engine_step(void* h, const smcl_cloud* scan, const smcl_odom* odo, smcl_frame_result* out) {
  return guard([&] {
    auto* e = static_cast<FilterEngine*>(h);
    OdometryInput o;
    o.delta = load_pose(odo->delta);
    std::memcpy(o.cov.m, odo->cov, 36 * sizeof(double));
    o.valid = odo->valid != 0;
    const FrameResult r = e->step(load_cloud(scan), o);
    std::memset(out, 0, sizeof(*out));
    store_pose(r.representative, out->representative);
    out->rep_log_post = r.rep_log_post;
    out->rep_index = r.rep_index;
    out->rep_id = r.rep_id;
    out->scan_empty = r.scan_empty;
    out->observation_rejected = r.observation_rejected;
    out->n_particles = static_cast<std::int64_t>(r.n_particles);
    out->mean_n_matched = r.mean_n_matched;
    out->predict_ms = r.times_ms[0];
    out->neighbor_ms = r.times_ms[1];
    out->likelihood_ms = r.times_ms[2];
    out->update_ms = r.times_ms[3];
    out->posterior_ms = r.times_ms[4];
    out->total_ms = r.times_ms[5];
    store_stats(r.neighbor_stats, &out->neighbor_stats);
  });
}
std::int64_t orc_engine_num_particles(void* h) {
  return static_cast<std::int64_t>(static_cast<FilterEngine*>(h)->particles().size());
}
int orc_engine_get(void* h, smcl_particles_view* view) {
  return guard([&] { store_set(static_cast<FilterEngine*>(h)->particles(), view); });
}
void orc_engine_set_frame(void* h, std::int64_t f) { static_cast<FilterEngine*>(h)->set_frame_index(f); }
int orc_engine_set(void* h, const smcl_particles_view* view) {
  return guard([&] { static_cast<FilterEngine*>(h)->particles() = load_set(view); });
}

}  // extern "C"
