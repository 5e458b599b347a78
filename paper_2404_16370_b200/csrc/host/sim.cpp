// Synthetic-world generator (the reference's sim/world.cpp: analytic
// rectangle worlds, surface sampling, ray-cast scans). Workload input for
// tests and bench.py; not part of the per-frame hot path.
#include <cmath>
#include <stdexcept>
#include <vector>

#include "../smcl_math.cuh"
#include "prep.hpp"
#include "sim.hpp"

namespace smcl::host {

namespace {
inline void cross(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
inline double dot3(const double a[3], const double b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

void push(std::vector<Rect>& w, double ox, double oy, double oz, double ux, double uy, double uz, double vx, double vy,
          double vz) {
  w.push_back({{ox, oy, oz}, {ux, uy, uz}, {vx, vy, vz}});
}
}  // namespace

// world.cpp:51-60
void add_box(std::vector<Rect>& w, const double lo[3], const double hi[3]) {
  const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  push(w, lo[0], lo[1], lo[2], dx, 0, 0, 0, dy, 0);
  push(w, lo[0], lo[1], hi[2], dx, 0, 0, 0, dy, 0);
  push(w, lo[0], lo[1], lo[2], dx, 0, 0, 0, 0, dz);
  push(w, lo[0], hi[1], lo[2], dx, 0, 0, 0, 0, dz);
  push(w, lo[0], lo[1], lo[2], 0, dy, 0, 0, 0, dz);
  push(w, hi[0], lo[1], lo[2], 0, dy, 0, 0, 0, dz);
}

// world.cpp:62-75
void add_wall_y(std::vector<Rect>& w, double y, double x0, double x1, double z0, double z1, double dx0, double dx1,
                double dh) {
  auto rect = [&](double a0, double a1, double b0, double b1) {
    if (a1 - a0 <= 1e-9 || b1 - b0 <= 1e-9) return;
    push(w, a0, y, b0, a1 - a0, 0, 0, 0, 0, b1 - b0);
  };
  if (dx1 <= dx0 || dh <= z0) {
    rect(x0, x1, z0, z1);
    return;
  }
  rect(x0, dx0, z0, z1);
  rect(dx1, x1, z0, z1);
  rect(dx0, dx1, dh, z1);
}

// world.cpp:77-133
std::vector<Rect> corridor_world(const CorridorSpec& s) {
  if (s.n_rooms < 1) throw std::invalid_argument("corridor_world: need at least one room");
  std::vector<Rect> w;
  const double h = s.height, len = s.corridor_length, cw = s.corridor_width, pitch = len / s.n_rooms;
  push(w, 0, 0, 0, len, 0, 0, 0, cw, 0);
  push(w, 0, 0, h, len, 0, 0, 0, cw, 0);
  add_wall_y(w, 0.0, 0.0, len, 0.0, h, 0, 0, 0);
  push(w, 0, 0, 0, 0, cw, 0, 0, 0, h);
  push(w, len, 0, 0, 0, cw, 0, 0, 0, h);
  double wall_x = 0.0;
  for (int r = 0; r < s.n_rooms; ++r) {
    const double cx = (r + 0.5) * pitch;
    const double dx0 = cx - 0.5 * s.door_width, dx1 = cx + 0.5 * s.door_width;
    add_wall_y(w, cw, wall_x, dx0, 0.0, h, 0, 0, 0);
    add_wall_y(w, cw, dx0, dx1, s.door_height, h, 0, 0, 0);
    wall_x = dx1;
  }
  add_wall_y(w, cw, wall_x, len, 0.0, h, 0, 0, 0);
  if (s.furniture) {
    const double stations[6] = {0.08, 0.22, 0.43, 0.58, 0.77, 0.93};
    const double widths[6] = {1.2, 0.7, 1.0, 0.5, 1.4, 0.8};
    const double depths[6] = {0.8, 0.5, 0.6, 0.9, 0.5, 0.7};
    const double heights[6] = {0.9, 1.4, 0.7, 1.1, 0.8, 1.3};
    for (int b = 0; b < 6; ++b) {
      const double cx = stations[b] * len;
      const double lo[3] = {std::max(0.2, cx - 0.5 * widths[b]), 0.0, 0.0};
      const double hi[3] = {std::min(len - 0.2, cx + 0.5 * widths[b]), depths[b], heights[b]};
      add_box(w, lo, hi);
    }
  }
  for (int r = 0; r < s.n_rooms; ++r) {
    const double cx = (r + 0.5) * pitch;
    const double rx0 = cx - 0.5 * s.room_width, rx1 = cx + 0.5 * s.room_width;
    const double ry0 = cw, ry1 = cw + s.room_depth;
    push(w, rx0, ry0, 0, rx1 - rx0, 0, 0, 0, ry1 - ry0, 0);
    push(w, rx0, ry0, h, rx1 - rx0, 0, 0, 0, ry1 - ry0, 0);
    add_wall_y(w, ry1, rx0, rx1, 0.0, h, 0, 0, 0);
    push(w, rx0, ry0, 0, 0, ry1 - ry0, 0, 0, 0, h);
    push(w, rx1, ry0, 0, 0, ry1 - ry0, 0, 0, 0, h);
  }
  return w;
}

std::vector<Rect> box_room(const double size[3]) {  // world.cpp:135-139
  std::vector<Rect> w;
  const double lo[3] = {0, 0, 0};
  add_box(w, lo, size);
  return w;
}

static double rect_area(const Rect& r) {
  double c[3];
  cross(r.u, r.v, c);
  return std::sqrt(dot3(c, c));
}

// world.cpp:140-160: round(area*density) uniform samples per rectangle.
std::vector<V3> sample_world_points(const std::vector<Rect>& w, double density, std::uint64_t seed) {
  if (w.empty()) throw std::invalid_argument("sample_world: empty world spec");
  if (!(density > 0.0)) throw std::invalid_argument("sample_world: density must be positive");
  std::vector<V3> pts;
  smcl::SplitMix64 rng(seed);
  for (const Rect& r : w) {
    const long long count = std::llround(rect_area(r) * density);
    for (long long i = 0; i < count; ++i) {
      const double u = rng.uniform01();
      const double v = rng.uniform01();
      pts.push_back({(r.o[0] + u * r.u[0]) + v * r.v[0], (r.o[1] + u * r.u[1]) + v * r.v[1],
                     (r.o[2] + u * r.u[2]) + v * r.v[2]});
    }
  }
  return pts;
}

// world.cpp:28-49
static bool raycast(const std::vector<Rect>& w, const double org[3], const double dir[3], double max_range,
                    double& out) {
  double best = max_range;
  bool hit = false;
  for (const Rect& r : w) {
    double n[3];
    cross(r.u, r.v, n);
    const double denom = dot3(dir, n);
    if (std::fabs(denom) < 1e-12) continue;
    const double ro[3] = {r.o[0] - org[0], r.o[1] - org[1], r.o[2] - org[2]};
    const double t = dot3(ro, n) / denom;
    if (t <= 1e-9 || t >= best) continue;
    const double q[3] = {(org[0] + t * dir[0]) - r.o[0], (org[1] + t * dir[1]) - r.o[1], (org[2] + t * dir[2]) - r.o[2]};
    const double u = dot3(q, r.u) / dot3(r.u, r.u);
    const double v = dot3(q, r.v) / dot3(r.v, r.v);
    if (u < 0.0 || u > 1.0 || v < 0.0 || v > 1.0) continue;
    best = t;
    hit = true;
  }
  out = best;
  return hit;
}

// world.cpp:162-181: points in the sensor frame.
std::vector<V3> simulate_scan(const std::vector<Rect>& w, const double pose[12], const SensorSpec& s,
                              std::uint64_t& rng_state) {
  std::vector<V3> hits;
  smcl::SplitMix64 rng(rng_state);
  for (int e = 0; e < s.n_elevations; ++e) {
    const double elev = s.elevations_deg[e] * kPi / 180.0;
    for (int a = 0; a < s.n_azimuth; ++a) {
      const double az = 2.0 * kPi * a / s.n_azimuth;
      const double ds[3] = {std::cos(elev) * std::cos(az), std::cos(elev) * std::sin(az), std::sin(elev)};
      double dw[3];
      for (int i = 0; i < 3; ++i) dw[i] = (pose[i * 3 + 0] * ds[0] + pose[i * 3 + 1] * ds[1]) + pose[i * 3 + 2] * ds[2];
      const double org[3] = {pose[9], pose[10], pose[11]};
      double range;
      const bool hit = raycast(w, org, dw, s.max_range, range);
      double noise = 0.0;
      if (s.noise_sigma > 0.0) {
        double z0, z1;
        rng.normal_pair(z0, z1);
        noise = s.noise_sigma * z0;
      }
      if (!hit) continue;
      const double r = range + noise;
      if (r < s.min_range) continue;
      hits.push_back({r * ds[0], r * ds[1], r * ds[2]});
    }
  }
  rng_state = rng.state;
  return hits;
}

}  // namespace smcl::host
