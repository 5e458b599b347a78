// Synthetic worlds (reference sim/world.hpp:15-85) for workload generation.
#pragma once

#include <cstdint>
#include <vector>

#include "prep.hpp"

namespace smcl::host {

struct Rect {
  double o[3], u[3], v[3];  // origin, edge_u, edge_v
};

struct CorridorSpec {
  double corridor_length = 40.0, corridor_width = 3.0, height = 3.0;
  int n_rooms = 4;
  double room_width = 6.0, room_depth = 5.0, door_width = 1.2, door_height = 2.2;
  bool furniture = true;
};

struct SensorSpec {
  int n_azimuth = 16;
  int n_elevations = 5;
  double elevations_deg[64] = {-30.0, -10.0, 0.0, 10.0, 30.0};
  double max_range = 30.0, min_range = 0.2, noise_sigma = 0.01;
};

void add_box(std::vector<Rect>& w, const double lo[3], const double hi[3]);
void add_wall_y(std::vector<Rect>& w, double y, double x0, double x1, double z0, double z1, double dx0, double dx1,
                double dh);
std::vector<Rect> corridor_world(const CorridorSpec& s);
std::vector<Rect> box_room(const double size[3]);
std::vector<V3> sample_world_points(const std::vector<Rect>& w, double density, std::uint64_t seed);
std::vector<V3> simulate_scan(const std::vector<Rect>& w, const double pose[12], const SensorSpec& s,
                              std::uint64_t& rng_state);

}  // namespace smcl::host
