// Host-only part of the C ABI (include/smcl_gpu.h): map/scan preparation and
// the synthetic-world generator. Compiled by the host compiler with OpenMP.
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/smcl_gpu.h"
#include "prep.hpp"
#include "sim.hpp"

namespace smcl {
extern thread_local std::string g_last_error;
}

using namespace smcl::host;

namespace {
template <class F>
int hguard(F&& f) {
  try {
    f();
    return SMCL_OK;
  } catch (const std::invalid_argument& e) {
    smcl::g_last_error = e.what();
    return SMCL_EINVAL;
  } catch (const std::logic_error& e) {
    smcl::g_last_error = e.what();
    return SMCL_ELOGIC;
  } catch (const std::exception& e) {
    smcl::g_last_error = e.what();
    return SMCL_ERUNTIME;
  }
}
const V3* as_v3(const double* p) { return reinterpret_cast<const V3*>(p); }

std::vector<Rect> load_rects(const double* r, int32_t n) {
  std::vector<Rect> w(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) std::memcpy(&w[static_cast<size_t>(i)], r + 9 * i, 9 * sizeof(double));
  return w;
}
int store_rects(const std::vector<Rect>& w, double* out, int32_t max_rects, int32_t* n_out) {
  *n_out = static_cast<int32_t>(w.size());
  if (out) {
    if (static_cast<int32_t>(w.size()) > max_rects) throw std::invalid_argument("rect buffer too small");
    for (size_t i = 0; i < w.size(); ++i) std::memcpy(out + 9 * i, &w[i], 9 * sizeof(double));
  }
  return SMCL_OK;
}
}  // namespace

extern "C" {

int smcl_estimate_covariances(const double* points, int64_t n, int k, double eps, double* sigma_out) {
  return hguard([&] { estimate_covariances(as_v3(points), n, k, eps, sigma_out); });
}

int smcl_downsample_to(const double* points, int64_t n, int64_t max_points, double leaf, double* out, int64_t* n_out) {
  return hguard([&] {
    const auto v = downsample_to(as_v3(points), n, static_cast<size_t>(max_points), leaf);
    std::memcpy(out, v.data(), v.size() * sizeof(V3));
    *n_out = static_cast<int64_t>(v.size());
  });
}

// filter.cpp:86-100
int smcl_make_scan_cloud(const double* points, int64_t n, const smcl_config* cfg, double* mu_out, double* sigma_out,
                         int64_t* n_out) {
  return hguard([&] {
    *n_out = 0;
    if (n < static_cast<int64_t>(cfg->covariance_k) + 1 || n < 5) return;
    const auto down = downsample_to(as_v3(points), n, static_cast<size_t>(cfg->n_scan_max), cfg->scan_voxel_leaf);
    const int k = std::min<int>(cfg->covariance_k, static_cast<int>(down.size()) - 1);
    if (k < 4) return;
    estimate_covariances(down.data(), static_cast<int64_t>(down.size()), k, cfg->epsilon_plane, sigma_out);
    std::memcpy(mu_out, down.data(), down.size() * sizeof(V3));
    const double nv = cfg->sensor_noise_sigma * cfg->sensor_noise_sigma;
    if (nv > 0.0)
      for (size_t i = 0; i < down.size(); ++i)
        for (int d = 0; d < 3; ++d) sigma_out[9 * i + 4 * d] = sigma_out[9 * i + 4 * d] + nv;
    *n_out = static_cast<int64_t>(down.size());
  });
}

int smcl_build_nnf(const smcl_cloud* map, double resolution, double padding, double max_query_dist, int32_t dims[3],
                   double origin[3], int32_t* cells) {
  return hguard([&] {
    if (!map || map->n <= 0) throw std::invalid_argument("build_nnf: empty map");
    Aabb b;
    if (map->bounds) {
      for (int a = 0; a < 3; ++a) {
        b.min[a] = map->bounds[a];
        b.max[a] = map->bounds[3 + a];
      }
    } else {
      b = compute_bounds(as_v3(map->mu), map->n);
    }
    const NnfGeometry g = nnf_geometry(b, resolution, padding, max_query_dist, size_t(1) << 30);
    for (int a = 0; a < 3; ++a) {
      dims[a] = g.dims[a];
      origin[a] = g.origin[a];
    }
    if (cells) build_nnf_cells(as_v3(map->mu), map->n, g, cells);
  });
}

void smcl_sim_default_corridor(smcl_corridor_spec* s) {
  const CorridorSpec d;
  s->corridor_length = d.corridor_length;
  s->corridor_width = d.corridor_width;
  s->height = d.height;
  s->n_rooms = d.n_rooms;
  s->furniture = d.furniture ? 1 : 0;
  s->room_width = d.room_width;
  s->room_depth = d.room_depth;
  s->door_width = d.door_width;
  s->door_height = d.door_height;
}

void smcl_sim_default_sensor(smcl_sensor_spec* s) {
  const SensorSpec d;
  std::memset(s, 0, sizeof(*s));
  s->n_azimuth = d.n_azimuth;
  s->n_elevations = d.n_elevations;
  for (int i = 0; i < d.n_elevations; ++i) s->elevations_deg[i] = d.elevations_deg[i];
  s->max_range = d.max_range;
  s->min_range = d.min_range;
  s->noise_sigma = d.noise_sigma;
}

int smcl_sim_corridor_world(const smcl_corridor_spec* spec, double* rects, int32_t max_rects, int32_t* n_rects) {
  return hguard([&] {
    CorridorSpec s;
    s.corridor_length = spec->corridor_length;
    s.corridor_width = spec->corridor_width;
    s.height = spec->height;
    s.n_rooms = spec->n_rooms;
    s.furniture = spec->furniture != 0;
    s.room_width = spec->room_width;
    s.room_depth = spec->room_depth;
    s.door_width = spec->door_width;
    s.door_height = spec->door_height;
    store_rects(corridor_world(s), rects, max_rects, n_rects);
  });
}

int smcl_sim_box_room(const double size[3], double* rects, int32_t max_rects, int32_t* n_rects) {
  return hguard([&] { store_rects(box_room(size), rects, max_rects, n_rects); });
}

int smcl_sim_sample_world(const double* rects, int32_t n_rects, double density, uint64_t seed, int cov_k, double eps,
                          double* mu_out, double* sigma_out, int64_t* n_out) {
  return hguard([&] {
    const auto pts = sample_world_points(load_rects(rects, n_rects), density, seed);
    *n_out = static_cast<int64_t>(pts.size());
    if (!mu_out) return;
    if (pts.size() < static_cast<size_t>(cov_k) + 1)
      throw std::invalid_argument("sample_world: too few samples; raise the density");
    std::memcpy(mu_out, pts.data(), pts.size() * sizeof(V3));
    if (sigma_out) estimate_covariances(pts.data(), static_cast<int64_t>(pts.size()), cov_k, eps, sigma_out);
  });
}

int smcl_sim_scan(const double* rects, int32_t n_rects, const double pose[12], const smcl_sensor_spec* sensor,
                  uint64_t* rng_state, double* points_out, int64_t* n_out) {
  return hguard([&] {
    SensorSpec s;
    s.n_azimuth = sensor->n_azimuth;
    s.n_elevations = sensor->n_elevations;
    for (int i = 0; i < sensor->n_elevations && i < 64; ++i) s.elevations_deg[i] = sensor->elevations_deg[i];
    s.max_range = sensor->max_range;
    s.min_range = sensor->min_range;
    s.noise_sigma = sensor->noise_sigma;
    const auto hits = simulate_scan(load_rects(rects, n_rects), pose, s, *rng_state);
    std::memcpy(points_out, hits.data(), hits.size() * sizeof(V3));
    *n_out = static_cast<int64_t>(hits.size());
  });
}

}  // extern "C"
